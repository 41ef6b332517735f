#!/bin/bash
for i in 1 2 3; do for lb in 2 3; do
  GPUAR_ROWS_LOG2_BLOCK=$lb timeout 300 python bench.py --steps 300 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; r=json.loads(sys.stdin.read()); print('lb=$lb', '%.4g'%r['value'], 'sel %.0f GB/s'%r['roofline']['achieved'], r['clocks']['sm_mhz'], r['clocks']['reasons'])"
done; done
