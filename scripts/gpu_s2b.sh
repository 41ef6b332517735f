#!/bin/bash
# Session 2: argmin row kernel v2 v3 (leftover calls in one predicated step).
mkdir -p gpurun_out/s2b
timeout 900 python -m pytest tests -m gpu -x -q -k "argmin or rows or smoke" > gpurun_out/s2b/gpu_tests.log 2>&1
tail -2 gpurun_out/s2b/gpu_tests.log
timeout 300 python bench.py --config c4 --rule argmin --steps 20 --no-e2e --no-cpu > gpurun_out/s2b/c4_argmin.json 2>&1
tail -1 gpurun_out/s2b/c4_argmin.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_rows" -s 3 -c 1 -o gpurun_out/s2b/prof_c4am python bench.py --config c4 --rule argmin --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/s2b/ncu_c4am.log 2>&1
