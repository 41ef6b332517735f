#!/bin/bash
# Session 2: lane loop with two Philox calls per round for p <= 1/4 (A/B vs HEAD), full GPU suite.
mkdir -p gpurun_out/s2y
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/s2y/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/s2y/gpu_tests.log
bash scripts/gpu_abn.sh s2y "base default" "--config c3 --dist exponential --M 1000 --steps 20|c3e3" "--config c3 --dist exponential --M 10000 --steps 20|c3e4" "--config c3 --dist exponential --M 100000 --steps 20|c3e5" "--config c3 --dist uniform --M 10000 --steps 20|c3u4" "--config c3 --dist pareto --M 1000 --steps 20|c3p3" "--config c1 --steps 300|c1"
for g in 1 2; do GPUAR_TEAM=$g timeout 300 python bench.py --config c3 --dist exponential --M 100000 --steps 20 --no-cpu --no-e2e > gpurun_out/s2y/c3e5_g$g.json 2>&1; echo "c3e5 forced g=$g $(python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'])" gpurun_out/s2y/c3e5_g$g.json)"; done
for g in 1 2 4; do GPUAR_TEAM=$g timeout 300 python bench.py --config c3 --dist pareto --M 1000 --steps 20 --no-cpu --no-e2e > gpurun_out/s2y/c3p3_g$g.json 2>&1; echo "c3p3 forced g=$g $(python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'])" gpurun_out/s2y/c3p3_g$g.json)"; done
