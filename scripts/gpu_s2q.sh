#!/bin/bash
# Session 2: programmatic dependent launch of the shared-vector kernel (A/B vs HEAD).
mkdir -p gpurun_out/s2q
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s2q/gpu_tests.log 2>&1
tail -2 gpurun_out/s2q/gpu_tests.log
bash scripts/gpu_abn.sh s2q "base default" "--config c1 --steps 300|c1" "--config c2 --steps 300|c2" "--config c3 --dist uniform --M 10000 --steps 20|c3u4" "--config c3 --dist exponential --M 10000 --steps 20|c3e4" "--config c3 --dist pareto --M 10000 --steps 20|c3p4"
for f in gpurun_out/s2q/c1_*_1.json gpurun_out/s2q/c2_*_1.json; do python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d.get('graph_steady_state'))" $f; done
