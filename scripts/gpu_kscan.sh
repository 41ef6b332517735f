#!/bin/bash
# Shared-vector kernel: throughput vs K (fixed overhead vs per-selection cost).
mkdir -p gpurun_out/kscan
for K in 1048576 4194304 16777216; do
  for d in uniform exponential; do
    timeout 200 python bench.py --config c3 --dist $d --M 1000 --K $K --steps 20 --no-e2e --no-cpu > gpurun_out/kscan/c3_${d}_$K.json 2>&1
  done
  timeout 200 python bench.py --config c2 --K $K --steps 50 --no-e2e --no-cpu > gpurun_out/kscan/c2_$K.json 2>&1
done
timeout 200 python bench.py --config c2 --steps 300 --no-e2e --no-cpu > gpurun_out/kscan/c2_65536.json 2>&1
python - <<'PY'
import json,glob
for p in sorted(glob.glob('gpurun_out/kscan/*.json')):
    try:
        l=[x for x in open(p).read().splitlines() if x.startswith('{')][-1]; r=json.loads(l)
        print(p.split('/')[-1], '%.3g'%r['value'], r['ms_per_step'], '%.3f'%r['roofline']['frac'])
    except Exception as e: print(p, 'ERR', open(p).read()[-300:])
PY
