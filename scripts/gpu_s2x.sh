#!/bin/bash
# Session 2: ncu --set full of the c5 shared-vector kernel (M = 1e6 Pareto, group-bound path).
mkdir -p gpurun_out/s2x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"select_shared" -s 1 -c 1 -o gpurun_out/s2x/prof_c5 python bench.py --config c5 --steps 1 --warmup 3 --max-trials 16777216 --no-cpu --no-e2e > gpurun_out/s2x/ncu_c5.log 2>&1
ls -la gpurun_out/s2x
