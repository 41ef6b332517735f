#!/bin/bash
# Session 2: work-stealing set-up values from the host (A/B vs HEAD), full GPU suite.
mkdir -p gpurun_out/s2w
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/s2w/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/s2w/gpu_tests.log
bash scripts/gpu_abn.sh s2w "base default" "--config c1 --steps 300|c1" "--config c2 --steps 300|c2" "--config c3 --dist uniform --M 10000 --steps 20|c3u4" "--config c3 --dist exponential --M 10000 --steps 20|c3e4" "--config c3 --dist pareto --M 1000 --steps 20|c3p3"
