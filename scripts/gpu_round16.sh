#!/bin/bash
mkdir -p gpurun_out/r16
for pf in 0 1; do for g in 0 1 2 4 8 16; do
  for spec in "c2 --steps 300:c2" "c3 --dist pareto --M 10000 --steps 10:c3p4" "c3 --dist uniform --M 10000 --steps 20:c3u4" "c3 --dist exponential --M 10000 --steps 20:c3e4"; do
    args=${spec%%:*}; name=${spec##*:}
    GPUAR_NO_PREFETCH=$pf GPUAR_GRAB=$g timeout 300 python bench.py --config $args --no-cpu --no-e2e > gpurun_out/r16/${name}_pf${pf}_g$g.json 2>&1
  done
done; done
