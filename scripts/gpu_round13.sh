#!/bin/bash
mkdir -p gpurun_out/r13
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 1000 --no-e2e --no-cpu > gpurun_out/r13/c4.json 2>&1
timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --max-trials 16777216 --no-cpu --no-e2e > gpurun_out/r13/c5.json 2>&1
timeout 300 python bench.py --config c3 --dist pareto --M 100000 --steps 20 --no-cpu --no-e2e > gpurun_out/r13/c3p5.json 2>&1
timeout 300 python bench.py --config c3 --dist pareto --M 10000 --steps 20 --no-cpu --no-e2e > gpurun_out/r13/c3p4.json 2>&1
