#!/bin/bash
mkdir -p gpurun_out/r20
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --config s1 --steps 20 --no-cpu > gpurun_out/r20/s1.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ssa_kernel -s 3 -c 1 -o gpurun_out/prof_s1_v20 python bench.py --config s1 --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_s1_v20.log 2>&1
