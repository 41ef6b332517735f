#!/bin/bash
# Session 2: full ncu captures of the c4 argmin row kernel and the c3/c2 shared-vector kernel.
mkdir -p gpurun_out/s2a
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_rows" -s 3 -c 1 -o gpurun_out/s2a/prof_c4am python bench.py --config c4 --rule argmin --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/s2a/ncu_c4am.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_shared" -s 3 -c 1 -o gpurun_out/s2a/prof_c3e4 python bench.py --config c3 --dist exponential --M 10000 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/s2a/ncu_c3e4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_shared" -s 3 -c 1 -o gpurun_out/s2a/prof_c2 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/s2a/ncu_c2.log 2>&1
ls -la gpurun_out/s2a
