#!/bin/bash
mkdir -p gpurun_out/r11
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -5 gpurun_out/gpu_tests.log
for d in uniform exponential pareto; do timeout 300 python bench.py --config c3 --dist $d --M 100000 --steps 20 --no-cpu --no-e2e > gpurun_out/r11/c3_${d}_100000.json 2>&1; done
timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --max-trials 16777216 --no-cpu --no-e2e > gpurun_out/r11/c5.json 2>&1
timeout 300 python bench.py --steps 1000 --no-e2e > gpurun_out/r11/c4.json 2>&1
timeout 300 python bench.py --config p1 --steps 100 --no-cpu --no-e2e > gpurun_out/r11/p1.json 2>&1
