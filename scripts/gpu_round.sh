#!/bin/bash
# One GPU session: tests, benches, microkernel, ncu launch list + full capture.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
timeout 120 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1
timeout 120 python scripts/philox_peak.py > gpurun_out/philox_peak.json 2>&1
timeout 400 python bench.py > gpurun_out/bench_c4.json 2>gpurun_out/bench_c4.err
for c in c1 c2 c5; do timeout 300 python bench.py --config $c --steps 200 --no-cpu --no-e2e > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; done
for d in uniform exponential pareto; do timeout 300 python bench.py --config c3 --dist $d --M 10000 --steps 200 --no-cpu --no-e2e > gpurun_out/bench_c3_$d.json 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_rows -s 3 -c 1 -o gpurun_out/prof_c4 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_shared -s 3 -c 1 -o gpurun_out/prof_c2 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c2.log 2>&1
tail -3 gpurun_out/gpu_tests.log
