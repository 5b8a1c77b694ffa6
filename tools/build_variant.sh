#!/bin/bash
# Build a variant of the library with extra nvcc -D flags for some sources (default
# hs_blend.cu; SRC="hs_binning.cu hs_capi.cu" ... to pick others, all rebuilt with
# the same flags):
#   tools/build_variant.sh NAME -DHS_BWD_WARPS=1 -DHS_BWD_MINB=14
# Output: paper_2406_02720_b200/lib/variants/NAME/libhalfsplat_b200.so (experiments only).
set -e
NAME=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
P=$R/paper_2406_02720_b200
OUT=$P/lib/variants/$NAME
mkdir -p $OUT
SRCS=${SRC:-hs_blend.cu}
OBJS=$(ls $P/lib/obj/*.o)
NEW=""
: > $OUT/ptxas.log
for S in $SRCS; do
  O=$(basename $S .cu).o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -I $P/csrc -I $R/include --expt-relaxed-constexpr -Xptxas -v "$@" \
    -c $P/csrc/$S -o $OUT/$O 2>> $OUT/ptxas.log
  OBJS=$(echo "$OBJS" | grep -v "/$O\$")
  NEW="$NEW $OUT/$O"
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared --cudart static -o $OUT/libhalfsplat_b200.so $OBJS $NEW -ldl
grep -A2 "blend_fwd_kernel\|blend_bwd_kernelILb0" $OUT/ptxas.log | grep -E "Used|spill" | sed "s/^/$NAME: /" || true
