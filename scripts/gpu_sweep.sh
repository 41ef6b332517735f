#!/bin/bash
# correctness after the kernel refactor, then the row-kernel occupancy sweep and the
# shared-vector configs.
mkdir -p gpurun_out/sweep
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
for ws in "16 3" "16 2" "20 2" "24 2" "27 2" "12 4" "8 6" "24 1" "32 1"; do
  set -- $ws
  GPUAR_ROWS_WARPS=$1 GPUAR_ROWS_STAGES=$2 timeout 300 python bench.py --steps 300 --no-cpu --no-e2e > gpurun_out/sweep/c4_w$1_s$2.json 2>&1
done
for c in c1 c2; do timeout 300 python bench.py --config $c --steps 300 --no-cpu --no-e2e > gpurun_out/sweep/$c.json 2>&1; done
for d in uniform exponential pareto; do for M in 1000 10000 100000; do timeout 300 python bench.py --config c3 --dist $d --M $M --steps 20 --no-cpu --no-e2e > gpurun_out/sweep/c3_${d}_$M.json 2>&1; done; done
timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --max-trials 16777216 --no-cpu --no-e2e > gpurun_out/sweep/c5.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_shared -s 3 -c 1 -o gpurun_out/prof_c3p python bench.py --config c3 --dist pareto --M 10000 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c3p.log 2>&1
timeout 120 python scripts/philox_peak.py > gpurun_out/philox_peak.json 2>&1
