#!/bin/bash
# Tuning experiments: build lib/exp_<name>.so from the current sources with the shared-vector
# kernel restricted to one team mode (all|lane|warp) and given __launch_bounds__.
#   scripts/build_variant.sh <name> <mode> "<launch bounds>"
set -e
name=$1; mode=$2; lb=$3
R=$(cd "$(dirname "$0")/.." && pwd)
D=/tmp/gpuar_variant_$name
rm -rf $D; mkdir -p $D/a/b $D/include
cp $R/paper_1404_0027_b200/csrc/* $D/a/b/; cp $R/include/gpuar.h $D/include/
python3 - "$mode" "$D/a/b/kernels_select.cu" <<'PY'
import sys
mode, path = sys.argv[1], sys.argv[2]
s = open(path).read()
if mode != 'all':
    a = s.index("  if (g == 1u) {\n    if (fold)\n      lane_loop")
    b = s.index("  }\n}\n", a) + 4
    call = {"lane": "lane_loop<PATH, %s>(P, ts, sbase, amax, pl)", "warp": "warp_loop<PATH, %s>(P, ts, sbase, amax, pl)"}[mode]
    s = s[:a] + "  if (fold) " + call % "true" + "; else " + call % "false" + ";\n" + s[b:]
open(path, 'w').write(s)
PY
sed -i "s/__launch_bounds__(1024, 1) select_shared_kernel/__launch_bounds__($lb) select_shared_kernel/" $D/a/b/kernels_select.cu
cd $D/a/b
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -shared -Xcompiler -fPIC \
  -o $R/paper_1404_0027_b200/lib/exp_$name.so gpuar_api.cu kernels_misc.cu kernels_select.cu kernels_rows.cu \
  kernels_argmin.cu kernels_ssa.cu kernels_it.cu
echo built exp_$name
