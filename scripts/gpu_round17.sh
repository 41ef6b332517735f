#!/bin/bash
mkdir -p gpurun_out/r17
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 1000 --no-cpu --no-e2e > gpurun_out/r17/c4.json 2>&1
timeout 300 python bench.py --steps 1000 --no-cpu --no-e2e > gpurun_out/r17/c4b.json 2>&1
timeout 300 python bench.py --config c2 --steps 300 --no-cpu --no-e2e > gpurun_out/r17/c2.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_rows -s 3 -c 1 -o gpurun_out/prof_c4_v17 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c4_v17.log 2>&1
