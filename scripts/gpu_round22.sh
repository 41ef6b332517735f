#!/bin/bash
mkdir -p gpurun_out/r22
GPUAR_ROWS_TWO=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rows or c4" > gpurun_out/gpu_tests_two.log 2>&1
tail -2 gpurun_out/gpu_tests_two.log
for i in 1 2; do
timeout 300 python bench.py --steps 1000 --no-cpu --no-e2e > gpurun_out/r22/c4_one_$i.json 2>&1
GPUAR_ROWS_TWO=1 timeout 300 python bench.py --steps 1000 --no-cpu --no-e2e > gpurun_out/r22/c4_two_$i.json 2>&1
done
GPUAR_ROWS_TWO=1 timeout 600 ncu --set full --clock-control none -k regex:select_rows -s 3 -c 1 -o gpurun_out/prof_c4_two python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:select_rows -s 3 -c 1 -o gpurun_out/prof_c4_one python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
