#!/bin/bash
# Session 2: c4 row-pipeline geometry under the sustained power cap (1000 steps).
out=gpurun_out/s2zk; mkdir -p $out
for rep in 1 2; do for ws in "24 2" "20 2" "16 2" "32 1"; do set -- $ws
  GPUAR_ROWS_WARPS=$1 GPUAR_ROWS_STAGES=$2 timeout 300 python bench.py --steps 1000 --no-cpu --no-e2e > $out/c4_w$1_s$2_$rep.json 2>&1
  echo "rep$rep W=$1 S=$2 $(python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('%.4g' % d['value'], d['clocks']['sm_mhz'])" $out/c4_w$1_s$2_$rep.json)"
done; done
