#!/bin/bash
# Session 2: argmin rule on the matrix with four interleaved Philox calls per iteration, shared-vector argmin two per iteration (A/B vs HEAD).
mkdir -p gpurun_out/s2h
timeout 900 python -m pytest tests -m gpu -x -q -k "argmin" > gpurun_out/s2h/gpu_tests.log 2>&1
tail -2 gpurun_out/s2h/gpu_tests.log
bash scripts/gpu_abn.sh s2h "base default" "--config c4 --rule argmin --steps 20|c4am" "--config p1 --steps 100|p1" "--config c4 --steps 200|c4"
