#!/bin/bash
# Build a variant of the library with extra nvcc -D flags for one source (default
# hs_blend.cu; SRC=hs_binning.cu ... to pick another):
#   tools/build_variant.sh NAME -DHS_BWD_WARPS=1 -DHS_BWD_MINB=14
# Output: paper_2406_02720_b200/lib/variants/NAME/libhalfsplat_b200.so (experiments only).
set -e
NAME=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
P=$R/paper_2406_02720_b200
OUT=$P/lib/variants/$NAME
mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -I $P/csrc -I $R/include --expt-relaxed-constexpr -Xptxas -v "$@" \
  -c $P/csrc/${SRC:-hs_blend.cu} -o $OUT/variant.o 2> $OUT/ptxas.log
OBJ=$(basename ${SRC:-hs_blend.cu} .cu).o
OBJS=$(ls $P/lib/obj/*.o | grep -v "/$OBJ\$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared --cudart static -o $OUT/libhalfsplat_b200.so $OBJS $OUT/variant.o
grep -A2 "blend_fwd_kernel\|blend_bwd_kernelILb0" $OUT/ptxas.log | grep -E "Used|spill" | sed "s/^/$NAME: /"
