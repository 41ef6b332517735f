#!/bin/bash
# A/B: lib/exp_base.so (HEAD) vs the working-tree build, interleaved on one box.
#   bash scripts/gpu_ab.sh <outdir> "<config args>|<label>" ...
out=gpurun_out/$1; shift
mkdir -p $out
val() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('%.4g %.4g' % (d['value'], d['roofline']['frac']))" $1 2>/dev/null || echo fail; }
for spec in "$@"; do
  args=${spec%%|*}; name=${spec##*|}
  for rep in 1 2; do
    GPUAR_LIBRARY=paper_1404_0027_b200/lib/exp_base.so timeout 300 python bench.py $args --no-cpu --no-e2e > $out/${name}_base_$rep.json 2>&1
    timeout 300 python bench.py $args --no-cpu --no-e2e > $out/${name}_new_$rep.json 2>&1
    echo "$name rep$rep base $(val $out/${name}_base_$rep.json) new $(val $out/${name}_new_$rep.json)"
  done
done
