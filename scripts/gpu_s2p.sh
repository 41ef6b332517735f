#!/bin/bash
# Session 2: team-size model with the finish costs recalibrated (45 per finishing round) (A/B vs HEAD).
mkdir -p gpurun_out/s2p
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s2p/gpu_tests.log 2>&1
tail -2 gpurun_out/s2p/gpu_tests.log
bash scripts/gpu_abn.sh s2p "base default" "--config c1 --steps 300|c1" "--config c2 --steps 300|c2" "--config c3 --dist uniform --M 1000 --steps 20|c3u3" "--config c3 --dist exponential --M 1000 --steps 20|c3e3" "--config c3 --dist exponential --M 100000 --steps 20|c3e5" "--config c3 --dist pareto --M 1000 --steps 20|c3p3" "--config c3 --dist pareto --M 10000 --steps 20|c3p4" "--config c3 --dist exponential --M 10000 --steps 20|c3e4" "--config c3 --dist pareto --M 100000 --steps 5|c3p5"
for f in gpurun_out/s2p/*_default_1.json; do python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], (d.get('trials') or {}).get('team'))" $f; done
