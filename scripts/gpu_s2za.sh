#!/bin/bash
# Session 2: two-call lane loop with the team model bounded to E <= 128 (A/B vs HEAD), full GPU suite.
mkdir -p gpurun_out/s2za
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/s2za/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/s2za/gpu_tests.log
bash scripts/gpu_abn.sh s2za "base default" "--config c1 --steps 300|c1" "--config c2 --steps 300|c2" "--config c3 --dist uniform --M 10000 --steps 20|c3u4" "--config c3 --dist exponential --M 1000 --steps 20|c3e3" "--config c3 --dist exponential --M 10000 --steps 20|c3e4" "--config c3 --dist exponential --M 100000 --steps 20|c3e5" "--config c3 --dist pareto --M 1000 --steps 20|c3p3" "--config c3 --dist pareto --M 10000 --steps 20|c3p4" "--config c5 --steps 2 --warmup 3 --max-trials 16777216|c5"
