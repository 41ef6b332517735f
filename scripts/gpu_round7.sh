#!/bin/bash
mkdir -p gpurun_out/r7
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -5 gpurun_out/gpu_tests.log
timeout 200 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1
timeout 300 python bench.py --steps 1000 --no-cpu --no-e2e > gpurun_out/r7/c4.json 2>&1
for c in c2; do timeout 300 python bench.py --config $c --steps 300 --no-cpu --no-e2e > gpurun_out/r7/$c.json 2>&1; done
timeout 300 python bench.py --config c3 --dist pareto --M 10000 --steps 20 --no-cpu --no-e2e > gpurun_out/r7/c3p.json 2>&1
timeout 600 python bench.py --config s1 --steps 20 --no-cpu > gpurun_out/r7/s1.json 2>&1
timeout 300 python bench.py --steps 1000 --no-cpu --no-e2e > gpurun_out/r7/c4b.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_rows -s 3 -c 1 -o gpurun_out/prof_c4_v7 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c4_v7.log 2>&1
