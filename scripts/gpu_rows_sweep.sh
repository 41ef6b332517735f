#!/bin/bash
mkdir -p gpurun_out/rsweep
for ws in "24 2" "20 2" "16 2" "16 4" "20 4" "24 2"; do
  set -- $ws
  GPUAR_ROWS_WARPS=$1 GPUAR_ROWS_STAGES=$2 timeout 300 python bench.py --steps 300 --no-cpu --no-e2e > gpurun_out/rsweep/c4_w$1_s$2.json 2>&1
  python -c "
import json; l=[x for x in open('gpurun_out/rsweep/c4_w$1_s$2.json') if x.startswith('{')]
r=json.loads(l[-1]) if l else None
print('w$1 s$2', '%.4g'%r['value'] if r else open('gpurun_out/rsweep/c4_w$1_s$2.json').read()[-300:], r and r['ms_per_step'], r and r['clocks'])"
done
