#!/bin/bash
# Session 2: ncu --set full of the current shared-vector kernel on c3 uniform M=10^4 and c2.
mkdir -p gpurun_out/s2v
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_shared" -s 3 -c 1 -o gpurun_out/s2v/prof_c3u4 python bench.py --config c3 --dist uniform --M 10000 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/s2v/ncu_c3u4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_shared" -s 3 -c 1 -o gpurun_out/s2v/prof_c2 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/s2v/ncu_c2.log 2>&1
ls gpurun_out/s2v
