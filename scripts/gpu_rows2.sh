#!/bin/bash
mkdir -p gpurun_out/rows2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rows or c4 or argmin or host" > gpurun_out/rows2/tests.log 2>&1
tail -3 gpurun_out/rows2/tests.log
for i in 1 2; do
timeout 300 python bench.py --steps 300 --no-cpu --no-e2e > gpurun_out/rows2/c4_$i.json 2>&1
python -c "
import json; l=[x for x in open('gpurun_out/rows2/c4_$i.json') if x.startswith('{')]
r=json.loads(l[-1]) if l else None
print('c4', '%.4g'%r['value'] if r else open('gpurun_out/rows2/c4_$i.json').read()[-300:], r and r['ms_per_step'], r and r['roofline']['achieved'], r and r['roofline']['row_stats_stream_gbs'], r and r['clocks'])"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_rows -s 3 -c 1 -o gpurun_out/prof_c4_v18 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/rows2/ncu.log 2>&1
tail -2 gpurun_out/rows2/ncu.log
