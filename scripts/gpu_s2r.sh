#!/bin/bash
# Session 2: programmatic dependent launch also for the argmin-rule and inverse-transform kernels.
mkdir -p gpurun_out/s2r
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/s2r/gpu_tests.log 2>&1
tail -2 gpurun_out/s2r/gpu_tests.log
bash scripts/gpu_abn.sh s2r "base default" "--config p1 --steps 100|p1" "--config c2 --rule it --steps 300|c2it" "--config c3 --dist uniform --M 1000 --steps 20|c3u3" "--config c3 --dist exponential --M 1000 --steps 20|c3e3" "--config c3 --dist pareto --M 1000 --steps 20|c3p3"
