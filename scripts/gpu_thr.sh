#!/bin/bash
mkdir -p gpurun_out/thr
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/thr/gpu_tests.log 2>&1
tail -3 gpurun_out/thr/gpu_tests.log
run() { # tag args...
  tag=$1; shift
  timeout 300 python bench.py "$@" --no-e2e --no-cpu > gpurun_out/thr/$tag.json 2>&1
  python -c "
import json; l=[x for x in open('gpurun_out/thr/$tag.json') if x.startswith('{')]
r=json.loads(l[-1]) if l else None
print('$tag', '%.4g'%r['value'] if r else open('gpurun_out/thr/$tag.json').read()[-300:], r and r['ms_per_step'], r and '%.3f'%r['roofline']['frac'])"
}
run c1 --config c1 --steps 300
run c2 --config c2 --steps 300
run c2_24 --config c2 --K 16777216 --steps 5
for d in uniform exponential pareto; do for M in 1000 10000 100000; do run c3_${d}_$M --config c3 --dist $d --M $M --steps 20; done; done
run c3u_24 --config c3 --dist uniform --M 1000 --K 16777216 --steps 10
run c5 --config c5 --steps 3 --warmup 3 --max-trials 16777216
