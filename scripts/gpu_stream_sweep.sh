#!/bin/bash
# row pipeline streaming ceiling vs row-block size / ring depth / warps (row_stats_stream_gbs)
for cfg in "24 2 2" "24 2 0" "24 2 1" "24 2 3" "24 2 4" "24 1 2" "16 2 2" "32 1 2" "12 4 2"; do
  set -- $cfg
  GPUAR_ROWS_WARPS=$1 GPUAR_ROWS_STAGES=$2 GPUAR_ROWS_LOG2_BLOCK=$3 timeout 300 python bench.py --steps 200 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; r=json.loads(sys.stdin.read()); print('W=$1 S=$2 lb=$3', '%.4g'%r['value'], 'sel %.0f GB/s'%r['roofline']['achieved'], 'stream %.0f GB/s'%r['roofline']['row_stats_stream_gbs'], r['clocks']['sm_mhz'])"
done
