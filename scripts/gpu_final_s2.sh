#!/bin/bash
# Session-2 close: the round-end evidence (scripts/gpu_final.sh) plus one ncu capture of the
# two-call lane loop (c3 exponential M = 10^4).
bash scripts/gpu_final.sh
mkdir -p gpurun_out/s2final
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_shared" -s 3 -c 1 -o gpurun_out/s2final/prof_c3e4 python bench.py --config c3 --dist exponential --M 10000 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/s2final/ncu_c3e4.log 2>&1
