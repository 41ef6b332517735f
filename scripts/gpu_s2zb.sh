#!/bin/bash
# Session 2: team sweep at c3 Pareto M = 10^4 (E ~ 292) after the two-call lane loop.
source /dev/null
out=gpurun_out/s2zb; mkdir -p $out
for g in 32 16 8 4 2; do
  GPUAR_TEAM=$g timeout 300 python bench.py --config c3 --dist pareto --M 10000 --steps 20 --no-cpu --no-e2e > $out/c3p4_g$g.json 2>&1
  echo "c3p4 g=$g $(python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'])" $out/c3p4_g$g.json)"
done
