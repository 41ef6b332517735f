#!/bin/bash
# Session 2: s1 timing variance -- repeated bench runs and an ncu launch list of ssa_kernel.
mkdir -p gpurun_out/s2j
for i in 1 2 3 4; do
  timeout 300 python bench.py --config s1 --steps 60 --no-cpu > gpurun_out/s2j/s1_$i.json 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('s1 run', sys.argv[2], '%.4g' % d['value'], d['ms_per_step'])" gpurun_out/s2j/s1_$i.json $i
done
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,smsp__inst_executed.sum --clock-control none -k regex:ssa_kernel --csv --log-file gpurun_out/s2j/ssa_launches.csv python bench.py --config s1 --steps 30 --warmup 3 --no-cpu > gpurun_out/s2j/ncu.log 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/s2j/ssa_launches.csv')) if len(r)>10]
hdr=rows[0]; ki=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ii=hdr.index('ID')
d={}
for r in rows[1:]:
    d.setdefault(r[ii],{})[r[ki]]=r[vi]
for k in sorted(d,key=int): print(k, d[k])
PY
