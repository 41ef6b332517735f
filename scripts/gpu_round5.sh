#!/bin/bash
mkdir -p gpurun_out/r5
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -5 gpurun_out/gpu_tests.log
for lb in 0 1 2 3 5; do GPUAR_ROWS_LOG2_BLOCK=$lb timeout 300 python bench.py --steps 1000 --no-cpu --no-e2e > gpurun_out/r5/c4_lb$lb.json 2>&1; done
GPUAR_ROWS_LOG2_BLOCK=0 timeout 300 python bench.py --steps 1000 --no-cpu --no-e2e > gpurun_out/r5/c4_lb0b.json 2>&1
GPUAR_ROWS_LOG2_BLOCK=2 timeout 300 python bench.py --steps 1000 --no-cpu --no-e2e > gpurun_out/r5/c4_lb2b.json 2>&1
timeout 600 python bench.py --config s1 --steps 20 > gpurun_out/r5/s1.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ssa_kernel -s 3 -c 1 -o gpurun_out/prof_s1 python bench.py --config s1 --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_s1.log 2>&1
