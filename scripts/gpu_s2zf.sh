#!/bin/bash
# Session 2: shared-vector CTA size sweep (GPUAR_SH_BLOCK) after PDL and the two-call lane loop.
out=gpurun_out/s2zf; mkdir -p $out
val() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('%.4g' % d['value'])" $1 2>/dev/null || echo fail; }
for spec in "--config c1 --steps 300|c1" "--config c2 --steps 300|c2" "--config c3 --dist uniform --M 10000 --steps 20|c3u4" "--config c3 --dist exponential --M 10000 --steps 20|c3e4" "--config c3 --dist pareto --M 1000 --steps 20|c3p3" "--config c3 --dist pareto --M 10000 --steps 20|c3p4" "--config c3 --dist pareto --M 100000 --steps 5|c3p5" "--config c5 --steps 2 --warmup 3 --max-trials 16777216|c5"; do
  args=${spec%%|*}; name=${spec##*|}
  line="$name"
  for b in 0 512 1024; do
    GPUAR_SH_BLOCK=$b timeout 300 python bench.py $args --no-cpu --no-e2e > $out/${name}_b$b.json 2>&1
    line="$line | b=$b $(val $out/${name}_b$b.json)"
  done
  echo "$line"
done
