#!/bin/bash
# Session 2: lane_loop fast hand-out path, A/B vs HEAD.
mkdir -p gpurun_out/s2e
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s2e/gpu_tests.log 2>&1
tail -2 gpurun_out/s2e/gpu_tests.log
bash scripts/gpu_ab.sh s2e "--config c1 --steps 300|c1" "--config c3 --dist uniform --M 10000 --steps 20|c3u4" "--config c3 --dist exponential --M 10000 --steps 20|c3e4" "--config c3 --dist exponential --M 100000 --steps 20|c3e5" "--config c3 --dist uniform --M 1000 --steps 20|c3u3" "--config c2 --steps 300|c2"
