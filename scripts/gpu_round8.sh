#!/bin/bash
mkdir -p gpurun_out/r8
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -5 gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 1000 --no-cpu --no-e2e > gpurun_out/r8/c4.json 2>&1
timeout 300 python bench.py --steps 1000 --no-cpu --no-e2e > gpurun_out/r8/c4b.json 2>&1
GPUAR_ROWS_WARPS=32 GPUAR_ROWS_STAGES=1 timeout 300 python bench.py --steps 1000 --no-cpu --no-e2e > gpurun_out/r8/c4_w32s1.json 2>&1
timeout 300 python bench.py --config c2 --rule it --steps 300 --no-cpu --no-e2e > gpurun_out/r8/c2_it.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_rows -s 3 -c 1 -o gpurun_out/prof_c4_v8 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c4_v8.log 2>&1
timeout 1500 python scripts/table1.py --runs 10 --out gpurun_out/table1_r01.json > gpurun_out/table1.log 2>&1
