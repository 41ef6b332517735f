#!/bin/bash
# correctness, then every config's bench line (short), philox peak.
mkdir -p gpurun_out/all
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
timeout 400 python bench.py --steps 500 --no-cpu --no-e2e > gpurun_out/all/c4.json 2>&1
for c in c1 c2; do timeout 300 python bench.py --config $c --steps 300 --no-cpu --no-e2e > gpurun_out/all/$c.json 2>&1; done
for d in uniform exponential pareto; do for M in 1000 10000 100000; do timeout 300 python bench.py --config c3 --dist $d --M $M --steps 20 --no-cpu --no-e2e > gpurun_out/all/c3_${d}_$M.json 2>&1; done; done
timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --max-trials 16777216 --no-cpu --no-e2e > gpurun_out/all/c5.json 2>&1
timeout 120 python scripts/philox_peak.py > gpurun_out/philox_peak.json 2>&1
