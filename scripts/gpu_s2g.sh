#!/bin/bash
# Session 2: parallel team choice at CTA start-up (A/B vs HEAD), full GPU suite with the
# argmin row-shape parity test.
mkdir -p gpurun_out/s2g
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/s2g/gpu_tests.log 2>&1
tail -2 gpurun_out/s2g/gpu_tests.log
bash scripts/gpu_abn.sh s2g "base default" "--config c1 --steps 300|c1" "--config c2 --steps 300|c2" "--config c3 --dist uniform --M 10000 --steps 20|c3u4" "--config c3 --dist exponential --M 1000 --steps 20|c3e3" "--config c3 --dist pareto --M 1000 --steps 20|c3p3"
