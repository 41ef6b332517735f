#!/bin/bash
# round-end evidence: tests, smoke, default bench (full line), launch list, ncu full capture.
mkdir -p gpurun_out/r14
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
timeout 200 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r14/c4_default.json 2> gpurun_out/r14/c4_default.err
timeout 600 python bench.py --impl reference > gpurun_out/r14/ref_default.json 2> gpurun_out/r14/ref_default.err
for c in c1 c2; do timeout 300 python bench.py --config $c --steps 300 --no-e2e > gpurun_out/r14/$c.json 2>&1; done
timeout 300 python bench.py --config c3 --dist pareto --M 10000 --steps 20 --no-e2e > gpurun_out/r14/c3p4.json 2>&1
timeout 600 python bench.py --config s1 --steps 20 > gpurun_out/r14/s1.json 2>&1
timeout 300 python bench.py --config p1 --steps 100 --no-e2e > gpurun_out/r14/p1.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_final.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_rows -s 3 -c 1 -o gpurun_out/prof_c4_final python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c4_final.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_shared -s 3 -c 1 -o gpurun_out/prof_c2_final python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c2_final.log 2>&1
