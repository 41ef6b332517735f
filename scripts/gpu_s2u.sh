#!/bin/bash
# Session 2: argmin-rule shared-vector grid = one resident wave (A/B vs HEAD), full GPU suite.
mkdir -p gpurun_out/s2u
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/s2u/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/s2u/gpu_tests.log
bash scripts/gpu_abn.sh s2u "base default" "--config p1 --steps 100|p1" "--config p1 --M 64 --steps 100|p1m64" "--config p1 --M 256 --steps 100|p1m256"
