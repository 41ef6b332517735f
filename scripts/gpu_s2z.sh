#!/bin/bash
# Session 2: team model with the two-call lane loop (A/B vs HEAD = one call per round), full GPU suite.
mkdir -p gpurun_out/s2z
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/s2z/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/s2z/gpu_tests.log
bash scripts/gpu_abn.sh s2z "base default" "--config c3 --dist exponential --M 100000 --steps 20|c3e5" "--config c3 --dist pareto --M 1000 --steps 20|c3p3" "--config c3 --dist pareto --M 10000 --steps 20|c3p4" "--config c5 --steps 2 --warmup 3 --max-trials 16777216|c5" "--config c3 --dist uniform --M 1000 --steps 20|c3u3" "--config c2 --steps 300|c2"
for f in gpurun_out/s2z/*_default_1.json; do python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], (d.get('trials') or {}).get('team'))" $f; done
GPUAR_TEAM=32 timeout 300 python bench.py --config c3 --dist pareto --M 10000 --steps 20 --no-cpu --no-e2e > gpurun_out/s2z/c3p4_g32.json 2>&1; echo "c3p4 forced g=32 $(tail -c 2000 gpurun_out/s2z/c3p4_g32.json | python -c "import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])['value'])")"
