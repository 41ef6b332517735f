#!/bin/bash
mkdir -p gpurun_out/rows3
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/rows3/tests.log 2>&1
tail -2 gpurun_out/rows3/tests.log
for i in 1 2; do
timeout 300 python bench.py --steps 1000 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('c4', r['value'], r['roofline']['achieved'], r['roofline']['row_stats_stream_gbs'], r['clocks'])"
done
timeout 600 python bench.py --config s1 --steps 20 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('s1', r['value'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_rows -s 3 -c 1 -o gpurun_out/prof_c4_v19 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/rows3/ncu.log 2>&1
tail -1 gpurun_out/rows3/ncu.log
