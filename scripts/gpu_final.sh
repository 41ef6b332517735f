#!/bin/bash
# Round-end evidence: every workload's full bench line into gpurun_out/final.
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final/gpu_tests.log 2>&1
tail -3 gpurun_out/final/gpu_tests.log
timeout 200 python __graft_entry__.py --smoke > gpurun_out/final/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/final/c4.json 2> gpurun_out/final/c4.err
timeout 600 python bench.py --impl reference > gpurun_out/final/c4_reference.json 2>&1
timeout 300 python bench.py --config c1 --steps 300 > gpurun_out/final/c1.json 2>&1
timeout 300 python bench.py --config c2 --steps 300 > gpurun_out/final/c2.json 2>&1
for d in uniform exponential pareto; do for M in 1000 10000 100000; do timeout 300 python bench.py --config c3 --dist $d --M $M --steps 20 --no-e2e > gpurun_out/final/c3_${d}_$M.json 2>&1; done; done
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --max-trials 16777216 --no-e2e --cpu-seconds 20 > gpurun_out/final/c5.json 2>&1
timeout 300 python bench.py --config p1 --steps 100 > gpurun_out/final/p1.json 2>&1
timeout 300 python bench.py --config c4 --rule argmin --steps 20 --no-e2e > gpurun_out/final/c4_argmin.json 2>&1
timeout 300 python bench.py --config c2 --rule it --steps 300 --no-e2e > gpurun_out/final/c2_it.json 2>&1
timeout 600 python bench.py --config s1 --steps 20 > gpurun_out/final/s1.json 2>&1
timeout 120 python scripts/philox_peak.py > gpurun_out/final/philox_peak.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_c4_final.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/final/launches_c4.log 2>&1
python scripts/collect_results.py gpurun_out/final > gpurun_out/final/results.md
