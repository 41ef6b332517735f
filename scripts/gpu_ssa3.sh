#!/bin/bash
mkdir -p gpurun_out/ssa3
timeout 900 python -m pytest tests/test_gpu_ssa.py -m gpu -x -q > gpurun_out/ssa3/tests.log 2>&1
tail -3 gpurun_out/ssa3/tests.log
for i in 1 2; do
timeout 600 python bench.py --config s1 --steps 20 --no-cpu > gpurun_out/ssa3/s1_$i.json 2>&1
python -c "
import json; l=[x for x in open('gpurun_out/ssa3/s1_$i.json') if x.startswith('{')]
r=json.loads(l[-1]) if l else None
print('s1', '%.4g'%r['value'] if r else open('gpurun_out/ssa3/s1_$i.json').read()[-300:], r and r['ms_per_step'], r and r['clocks'])"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ssa_kernel -s 1 -c 1 -o gpurun_out/prof_s1_v23 python bench.py --config s1 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ssa3/ncu.log 2>&1
tail -1 gpurun_out/ssa3/ncu.log
