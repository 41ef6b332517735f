#!/bin/bash
# Session 2: shared-vector CTA-size policy (largest block within 3/4 of the best resident threads), A/B vs HEAD.
mkdir -p gpurun_out/s2zg
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/s2zg/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/s2zg/gpu_tests.log
bash scripts/gpu_abn.sh s2zg "base default" "--config c1 --steps 300|c1" "--config c2 --steps 300|c2" "--config c3 --dist uniform --M 1000 --steps 20|c3u3" "--config c3 --dist exponential --M 1000 --steps 20|c3e3" "--config c3 --dist pareto --M 10000 --steps 20|c3p4" "--config c2 --rule it --steps 300|c2it" "--config p1 --steps 100|p1"
