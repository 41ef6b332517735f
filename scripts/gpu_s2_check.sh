#!/bin/bash
# Session-2 re-entry check: GPU tests, smoke and the default bench line on a fresh box.
mkdir -p gpurun_out/s2v0
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/s2v0/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s2v0/gpu_tests.log 2>&1
tail -3 gpurun_out/s2v0/gpu_tests.log
timeout 200 python __graft_entry__.py --smoke > gpurun_out/s2v0/smoke.log 2>&1; echo smoke $?
timeout 600 python bench.py > gpurun_out/s2v0/c4.json 2> gpurun_out/s2v0/c4.err
cat gpurun_out/s2v0/c4.json
timeout 300 python bench.py --config c4 --rule argmin --steps 20 --no-e2e > gpurun_out/s2v0/c4_argmin.json 2>&1
tail -1 gpurun_out/s2v0/c4_argmin.json
