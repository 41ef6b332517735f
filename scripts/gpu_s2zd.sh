#!/bin/bash
# Session 2: final c4 argmin line after the batched leftovers (+ its ncu capture).
mkdir -p gpurun_out/s2zd
timeout 300 python bench.py --config c4 --rule argmin --steps 20 --no-e2e > gpurun_out/s2zd/c4_argmin.json 2>&1
tail -c 600 gpurun_out/s2zd/c4_argmin.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_rows" -s 3 -c 1 -o gpurun_out/s2zd/prof_c4am python bench.py --config c4 --rule argmin --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/s2zd/ncu_c4am.log 2>&1
