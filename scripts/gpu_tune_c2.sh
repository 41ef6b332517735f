#!/bin/bash
mkdir -p gpurun_out/tune
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/tune/parity.log 2>&1; tail -2 gpurun_out/tune/parity.log

run() { # tag env... -- args
  tag=$1; shift
  env "$@" timeout 200 python bench.py --config c2 --steps 300 --no-e2e --no-cpu > gpurun_out/tune/$tag.json 2>&1
  python -c "
import json; l=[x for x in open('gpurun_out/tune/$tag.json') if x.startswith('{')]
r=json.loads(l[-1]) if l else None
print('$tag', '%.4g'%r['value'] if r else open('gpurun_out/tune/$tag.json').read()[-300:], r and r['ms_per_step'])"
}
run base X=1
for g in 1 4 8 16; do run grab$g GPUAR_GRAB=$g; done
run nopf GPUAR_NO_PREFETCH=1
for c in 1 2 3; do run ctas$c GPUAR_SH_CTAS_PER_SM=$c; done
