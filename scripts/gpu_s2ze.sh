#!/bin/bash
# Session 2: c2 CTAs-per-SM sweep after PDL.
out=gpurun_out/s2ze; mkdir -p $out
for rep in 1 2; do for n in 0 4 3 2; do
  GPUAR_SH_CTAS_PER_SM=$n timeout 300 python bench.py --config c2 --steps 300 --no-cpu --no-e2e > $out/c2_n${n}_$rep.json 2>&1
  echo "c2 ctas/sm=$n rep$rep $(python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'])" $out/c2_n${n}_$rep.json)"
done; done
