#!/bin/bash
mkdir -p gpurun_out/r18
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
for c in c1 c2; do timeout 300 python bench.py --config $c --steps 300 --no-cpu --no-e2e > gpurun_out/r18/$c.json 2>&1; done
for d in uniform exponential pareto; do for M in 1000 10000 100000; do timeout 300 python bench.py --config c3 --dist $d --M $M --steps 20 --no-cpu --no-e2e > gpurun_out/r18/c3_${d}_$M.json 2>&1; done; done
timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --max-trials 16777216 --no-cpu --no-e2e > gpurun_out/r18/c5.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_shared" -s 3 -c 1 -o gpurun_out/prof_c2_v18 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c2_v18.log 2>&1
