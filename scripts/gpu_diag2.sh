#!/bin/bash
mkdir -p gpurun_out/diag
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "shared or c1 or c2 or c3 or c5 or stream or error or epoch" > gpurun_out/diag/parity.log 2>&1
tail -3 gpurun_out/diag/parity.log
timeout 120 python scripts/diag_fixed.py 1000 uniform > gpurun_out/diag/u1000.txt 2>&1
timeout 120 python scripts/diag_fixed.py 1029 yeast > gpurun_out/diag/y1029.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/diag/launches.csv python scripts/diag_fixed.py 1000 uniform > /dev/null 2>&1
cat gpurun_out/diag/u1000.txt gpurun_out/diag/y1029.txt
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/diag/launches.csv')))
hdr=next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
h=rows[hdr]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
seq=[(r[ki][:40], float(r[vi].replace(',',''))) for r in rows[hdr+1:] if len(r)>vi]
sel=[v for k,v in seq if 'select_shared' in k]
for i in range(0, len(sel), 405):
    ch=sel[i:i+405]
    print('K-stage', i//405, 'n', len(ch), 'median kernel ns', sorted(ch)[len(ch)//2])
PY
for c in c1 c2; do timeout 200 python bench.py --config $c --steps 300 --no-e2e --no-cpu > gpurun_out/diag/$c.json 2>&1; done
timeout 200 python bench.py --config c3 --dist uniform --M 1000 --steps 20 --no-e2e --no-cpu > gpurun_out/diag/c3u.json 2>&1
timeout 200 python bench.py --config c3 --dist pareto --M 100000 --steps 5 --no-e2e --no-cpu > gpurun_out/diag/c3p.json 2>&1
for f in c1 c2 c3u c3p; do python -c "
import json,sys; l=[x for x in open('gpurun_out/diag/$f.json') if x.startswith('{')][-1]; r=json.loads(l); print('$f', '%.4g'%r['value'], r['ms_per_step'], '%.3f'%r['roofline']['frac'])"; done
