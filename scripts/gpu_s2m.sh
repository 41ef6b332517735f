#!/bin/bash
# Session 2: s1 bench after warming torch's accumulate kernel outside the timed region.
mkdir -p gpurun_out/s2m
for i in 1 2 3; do
  timeout 600 python bench.py --config s1 --steps 20 > gpurun_out/s2m/s1_$i.json 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('s1 run', sys.argv[2], '%.4g' % d['value'], d['ms_per_step'], d['roofline']['frac'])" gpurun_out/s2m/s1_$i.json $i
done
