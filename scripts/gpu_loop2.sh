#!/bin/bash
mkdir -p gpurun_out/var
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/var/parity.log 2>&1
tail -3 gpurun_out/var/parity.log
L=paper_1404_0027_b200/lib
run() { # tag args...
  tag=$1; shift
  timeout 200 python bench.py "$@" --no-e2e --no-cpu > gpurun_out/var/$tag.json 2>&1
  python -c "
import json; l=[x for x in open('gpurun_out/var/$tag.json') if x.startswith('{')]
r=json.loads(l[-1]) if l else None
print('$tag', '%.4g'%r['value'] if r else open('gpurun_out/var/$tag.json').read()[-300:], r and r['ms_per_step'], r and '%.3f'%r['roofline']['frac'])"
}
for d in uniform exponential; do
  run c3${d:0:1}_20 --config c3 --dist $d --M 1000 --steps 20
  run c3${d:0:1}_24 --config c3 --dist $d --M 1000 --K 16777216 --steps 10
done
run c2_16 --config c2 --steps 300
run c2_24 --config c2 --K 16777216 --steps 5
run c3p4 --config c3 --dist pareto --M 10000 --steps 10
run c3p5 --config c3 --dist pareto --M 100000 --steps 5
run c1 --config c1 --steps 300
