#!/bin/bash
# A/B experiments: lib/exp_<name>.so from the working tree with kernels_select.cu compiled
# with -maxrregcount=<n> (the other files as usual); optionally from git revision <rev>.
#   scripts/build_select_maxreg.sh <name> <n> [rev]
set -e
name=$1; n=$2; rev=$3
R=$(cd "$(dirname "$0")/.." && pwd)
D=/tmp/gpuar_mr_$name; rm -rf $D; mkdir -p $D
S=$R
if [ -n "$rev" ]; then S=$D/src; mkdir -p $S; git -C $R archive $rev paper_1404_0027_b200/csrc include | tar -x -C $S; fi
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC"
cd $S/paper_1404_0027_b200/csrc
for f in gpuar_api kernels_misc kernels_rows kernels_argmin kernels_ssa kernels_it; do
  nvcc $F -c $f.cu -o $D/$f.o &
done
nvcc $F -maxrregcount=$n -Xptxas -v -c kernels_select.cu -o $D/kernels_select.o 2>&1 | grep -A1 "select_shared" | grep -E "Used|spill" &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/paper_1404_0027_b200/lib/exp_$name.so $D/*.o
echo built exp_$name
