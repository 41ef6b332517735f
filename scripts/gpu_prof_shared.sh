#!/bin/bash
for spec in "c3 --dist uniform --M 10000:c3u4" "c3 --dist exponential --M 10000:c3e4" "c2:c2"; do
  args=${spec%%:*}; name=${spec##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_shared" -s 3 -c 1 -o gpurun_out/prof_${name}_v19 python bench.py --config $args --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_${name}_v19.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3u4.csv python bench.py --config c3 --dist uniform --M 10000 --steps 5 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
