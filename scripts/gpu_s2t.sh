#!/bin/bash
# Session 2: cooperative drain phase in warp_loop (A/B vs HEAD).
mkdir -p gpurun_out/s2t
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/s2t/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/s2t/gpu_tests.log
bash scripts/gpu_abn.sh s2t "base default" "--config c2 --steps 300|c2" "--config c3 --dist pareto --M 10000 --steps 20|c3p4" "--config c3 --dist pareto --M 100000 --steps 5|c3p5" "--config c5 --steps 2 --warmup 3 --max-trials 16777216|c5"
