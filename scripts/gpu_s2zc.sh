#!/bin/bash
# Session 2: argmin rule on the matrix with the leftover calls batched over 16 rows (A/B vs HEAD).
mkdir -p gpurun_out/s2zc
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/s2zc/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/s2zc/gpu_tests.log
timeout 300 python scripts/sanitize_cases.py > gpurun_out/s2zc/sanitize_plain.log 2>&1; echo "sanitize cases rc=$?"
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/s2zc/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -1 gpurun_out/s2zc/memcheck.log
bash scripts/gpu_abn.sh s2zc "base default" "--config c4 --rule argmin --steps 20|c4am" "--config c4 --steps 200|c4"
