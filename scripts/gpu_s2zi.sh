#!/bin/bash
# Session 2 close: ncu --set full of the c4 row kernel as it ships (PDL launch) and of c2.
mkdir -p gpurun_out/s2zi
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_rows" -s 3 -c 1 -o gpurun_out/s2zi/prof_c4 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/s2zi/ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_shared" -s 3 -c 1 -o gpurun_out/s2zi/prof_c2 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/s2zi/ncu_c2.log 2>&1
ls gpurun_out/s2zi
