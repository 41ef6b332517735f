#!/bin/bash
# Session 2: PDL also for the statistics / thresholds / row kernels (A/B vs HEAD), with e2e.
mkdir -p gpurun_out/s2s
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/s2s/gpu_tests.log 2>&1
tail -2 gpurun_out/s2s/gpu_tests.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/s2s/smoke.log 2>&1; echo "smoke rc=$?"
v() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); e=d.get('e2e') or {}; print('%.4g e2e %s' % (d['value'], e.get('value')))" $1 2>/dev/null || echo fail; }
for rep in 1 2; do
  for lib in base default; do
    if [ $lib = default ]; then L=paper_1404_0027_b200/lib/libgpuar.so; else L=paper_1404_0027_b200/lib/exp_$lib.so; fi
    GPUAR_LIBRARY=$L timeout 300 python bench.py --config c2 --steps 300 --no-cpu > gpurun_out/s2s/c2_${lib}_$rep.json 2>&1
    GPUAR_LIBRARY=$L timeout 300 python bench.py --config c1 --steps 300 --no-cpu > gpurun_out/s2s/c1_${lib}_$rep.json 2>&1
    GPUAR_LIBRARY=$L timeout 600 python bench.py --steps 300 --no-cpu --no-e2e > gpurun_out/s2s/c4_${lib}_$rep.json 2>&1
    echo "rep$rep $lib c2 $(v gpurun_out/s2s/c2_${lib}_$rep.json) | c1 $(v gpurun_out/s2s/c1_${lib}_$rep.json) | c4 $(v gpurun_out/s2s/c4_${lib}_$rep.json)"
  done
done
