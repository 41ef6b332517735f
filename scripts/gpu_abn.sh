#!/bin/bash
# N-way A/B of in-tree builds, interleaved on one box:
#   bash scripts/gpu_abn.sh <outdir> "<lib1> <lib2> ..." "<config args>|<label>" ...
# (lib "default" = lib/libgpuar.so, else lib/exp_<lib>.so)
out=gpurun_out/$1; libs=$2; shift 2
mkdir -p $out
val() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('%.4g' % d['value'])" $1 2>/dev/null || echo fail; }
for spec in "$@"; do
  args=${spec%%|*}; name=${spec##*|}
  for rep in 1 2; do
    line="$name rep$rep"
    for lib in $libs; do
      if [ "$lib" = default ]; then L=paper_1404_0027_b200/lib/libgpuar.so; else L=paper_1404_0027_b200/lib/exp_$lib.so; fi
      GPUAR_LIBRARY=$L timeout 300 python bench.py $args --no-cpu --no-e2e > $out/${name}_${lib}_$rep.json 2>&1
      line="$line $lib $(val $out/${name}_${lib}_$rep.json)"
    done
    echo "$line"
  done
done
