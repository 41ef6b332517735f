#!/bin/bash
# Session 2: 1024-thread CTAs for the argmin-rule and inverse-transform kernels (A/B vs HEAD).
mkdir -p gpurun_out/s2zh
timeout 900 python -m pytest tests -m gpu -q -k "argmin or it_ or table1 or smoke" > gpurun_out/s2zh/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/s2zh/gpu_tests.log
bash scripts/gpu_abn.sh s2zh "base default" "--config p1 --steps 100|p1" "--config p1 --M 64 --steps 100|p1m64" "--config c2 --rule it --steps 300|c2it" "--config c3 --dist pareto --M 100000 --rule it --steps 50|c3p5it"
