#!/bin/bash
mkdir -p gpurun_out/diag
timeout 120 python scripts/diag_fixed.py 1000 uniform > gpurun_out/diag/u1000.txt 2>&1
timeout 120 python scripts/diag_fixed.py 1029 yeast > gpurun_out/diag/y1029.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/diag/launches.csv python scripts/diag_fixed.py 1000 uniform > /dev/null 2>&1
cat gpurun_out/diag/u1000.txt gpurun_out/diag/y1029.txt
python - <<'PY'
import csv
from collections import defaultdict
rows=list(csv.reader(open('gpurun_out/diag/launches.csv')))
hdr=next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
h=rows[hdr]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); gi=h.index('Grid Size') if 'Grid Size' in h else None
seq=[(r[ki][:40], float(r[vi].replace(',',''))) for r in rows[hdr+1:] if len(r)>vi]
# group consecutive runs of select kernels by K stage (each stage: 5+200+200 launches)
print(len(seq))
sel=[v for k,v in seq if 'select_shared' in k]
for i in range(0, len(sel), 405):
    ch=sel[i:i+405]
    print('K-stage', i//405, 'n', len(ch), 'median kernel ns', sorted(ch)[len(ch)//2])
PY
