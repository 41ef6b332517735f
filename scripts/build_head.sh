#!/bin/bash
# A/B experiments: build lib/exp_<name>.so from the sources of a git revision (default HEAD).
#   scripts/build_head.sh <name> [rev]
set -e
name=$1; rev=${2:-HEAD}
R=$(cd "$(dirname "$0")/.." && pwd)
D=/tmp/gpuar_rev_$name
rm -rf $D; mkdir -p $D
git -C $R archive $rev paper_1404_0027_b200/csrc include | tar -x -C $D
cd $D/paper_1404_0027_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -shared -Xcompiler -fPIC \
  -o $R/paper_1404_0027_b200/lib/exp_$name.so gpuar_api.cu kernels_misc.cu kernels_select.cu kernels_rows.cu \
  kernels_argmin.cu kernels_ssa.cu kernels_it.cu
echo built exp_$name from $rev
