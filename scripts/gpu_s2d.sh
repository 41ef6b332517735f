#!/bin/bash
# Session 2: shared-vector kernel with parameter-space Philox keys (A/B vs HEAD), argmin rows geometry.
mkdir -p gpurun_out/s2d
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s2d/gpu_tests.log 2>&1
tail -2 gpurun_out/s2d/gpu_tests.log
bash scripts/gpu_ab.sh s2d "--config c1 --steps 300|c1" "--config c2 --steps 300|c2" "--config c3 --dist uniform --M 10000 --steps 20|c3u4" "--config c3 --dist exponential --M 10000 --steps 20|c3e4" "--config c3 --dist pareto --M 10000 --steps 20|c3p4" "--config c5 --steps 2 --warmup 3 --max-trials 16777216|c5"
for wsp in "24 2" "32 1" "28 1" "20 2"; do set -- $wsp
  GPUAR_ROWS_WARPS=$1 GPUAR_ROWS_STAGES=$2 timeout 300 python bench.py --config c4 --rule argmin --steps 20 --no-e2e --no-cpu > gpurun_out/s2d/c4am_w$1_s$2.json 2>&1
  echo "argmin W=$1 S=$2 $(python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])" gpurun_out/s2d/c4am_w$1_s$2.json)"
done
