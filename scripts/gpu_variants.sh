#!/bin/bash
# A/B of shared-vector kernel variants (scripts/build_variant.sh) on c2 / c3.
mkdir -p gpurun_out/var
L=paper_1404_0027_b200/lib
run() { # tag lib args...
  tag=$1; lib=$2; shift 2
  GPUAR_LIBRARY=$lib timeout 200 python bench.py "$@" --no-e2e --no-cpu > gpurun_out/var/$tag.json 2>&1
  python -c "
import json; l=[x for x in open('gpurun_out/var/$tag.json') if x.startswith('{')]
r=json.loads(l[-1]) if l else None
print('$tag', '%.4g'%r['value'] if r else open('gpurun_out/var/$tag.json').read()[-300:], r and r['ms_per_step'], r and '%.3f'%r['roofline']['frac'])"
}
for v in libgpuar exp_lane4 exp_lane6 exp_lane8; do
  for d in uniform exponential; do
    run c3${d:0:1}_20_$v $L/$v.so --config c3 --dist $d --M 1000 --steps 20
    run c3${d:0:1}_24_$v $L/$v.so --config c3 --dist $d --M 1000 --K 16777216 --steps 10
  done
done
for v in libgpuar exp_warp4 exp_warp6; do
  run c2_16_$v $L/$v.so --config c2 --steps 300
  run c2_24_$v $L/$v.so --config c2 --K 16777216 --steps 5
  run c3p4_$v $L/$v.so --config c3 --dist pareto --M 10000 --steps 10
done
