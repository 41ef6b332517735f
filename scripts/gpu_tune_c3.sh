#!/bin/bash
# c3 work-stealing grab size sweep (GPUAR_GRAB) and K=1024 fixed cost
run() { # tag env... -- args
  tag=$1; shift; envs=$1; shift
  env $envs timeout 200 python bench.py "$@" --no-e2e --no-cpu 2>&1 | tail -1 | python -c "
import json,sys; r=json.loads(sys.stdin.read()); g=r.get('graph_steady_state') or {}; print('$tag', '%.4g'%r['value'], '%.2f us'%(r['ms_per_step']*1e3), 'graph %.2f us'%g.get('us_per_call',0))"
}
for d in uniform exponential; do
  for g in 0 8 32 64 128 256 1024; do
    run "c3_${d}_grab$g" "GPUAR_GRAB=$g" --config c3 --dist $d --M 1000 --steps 50
  done
  run "c3_${d}_nopf" "GPUAR_NO_PREFETCH=1" --config c3 --dist $d --M 1000 --steps 50
done
for g in 0 4 16; do run "c2_grab$g" "GPUAR_GRAB=$g" --config c2 --steps 300; done
