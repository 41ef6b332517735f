#!/bin/bash
mkdir -p gpurun_out/r23
timeout 1500 python -m pytest tests -m gpu -x -q -k "argmin or table1 or smoke" > gpurun_out/gpu_tests_am.log 2>&1
tail -2 gpurun_out/gpu_tests_am.log
timeout 300 python bench.py --config p1 --steps 100 --no-cpu --no-e2e > gpurun_out/r23/p1.json 2>&1
timeout 300 python bench.py --config p1 --M 64 --steps 100 --no-cpu --no-e2e > gpurun_out/r23/p1_64.json 2>&1
timeout 300 python bench.py --config c4 --rule argmin --steps 20 --no-cpu --no-e2e > gpurun_out/r23/c4_argmin.json 2>&1
