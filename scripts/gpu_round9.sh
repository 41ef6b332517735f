#!/bin/bash
mkdir -p gpurun_out/san gpurun_out/r9
timeout 900 compute-sanitizer --tool synccheck --num-cuda-barriers 65536 --target-processes all --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/san/synccheck2.log 2>&1
echo "synccheck rc=$?" > gpurun_out/san/summary2.txt; tail -3 gpurun_out/san/synccheck2.log >> gpurun_out/san/summary2.txt
for spec in "c3 --dist uniform --M 1000:c3u1k" "c3 --dist exponential --M 10000:c3e10k" "p1:p1" "c1:c1"; do
  args=${spec%%:*}; name=${spec##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_shared|argmin_shared" -s 3 -c 1 -o gpurun_out/prof_$name python bench.py --config $args --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_$name.log 2>&1
done
timeout 300 python bench.py --config c2 --rule it --steps 300 --no-cpu --no-e2e > gpurun_out/r9/c2_it.json 2>&1
timeout 300 python bench.py --config c3 --dist pareto --M 100000 --rule it --steps 20 --no-cpu --no-e2e > gpurun_out/r9/c3p_it.json 2>&1
