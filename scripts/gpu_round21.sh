#!/bin/bash
mkdir -p gpurun_out/r21
timeout 1500 python -m pytest tests/test_gpu_ssa.py tests/test_gpu_parity.py -m gpu -x -q -k "ssa or dimer or immigration or yeast_network or chunked" > gpurun_out/gpu_tests_ssa.log 2>&1
tail -3 gpurun_out/gpu_tests_ssa.log
timeout 600 python bench.py --config s1 --steps 20 --no-cpu > gpurun_out/r21/s1.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ssa_kernel -s 3 -c 1 -o gpurun_out/prof_s1_v21 python bench.py --config s1 --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_s1_v21.log 2>&1
python scripts/sanitize_cases.py > gpurun_out/r21/san.log 2>&1; timeout 900 compute-sanitizer --tool racecheck python scripts/sanitize_cases.py > gpurun_out/r21/racecheck.log 2>&1; tail -2 gpurun_out/r21/racecheck.log
