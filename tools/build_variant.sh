#!/bin/bash
# Build an experiment variant of the library: tools/build_variant.sh NAME "NVCC FLAGS" [source.cu ...]
# (default source: attn_bwd_tc.cu).  Output: ab_libs/NAME/libmugv_b200.so (git-ignored; travels with gpurun).
set -e
NAME=$1; FLAGS=$2; shift 2
SRCS=${@:-attn_bwd_tc.cu}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_2510_17519_b200/csrc
make -s -C $C -j16
OUT=$ROOT/ab_libs/$NAME; mkdir -p $OUT/obj
OBJS=""
for f in $C/_obj/*.o; do
  b=$(basename $f .o)
  if echo " $SRCS " | grep -q " $b.cu "; then
    nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
      -I$C -I$ROOT/include $FLAGS -c $C/$b.cu -o $OUT/obj/$b.o
    OBJS="$OBJS $OUT/obj/$b.o"
  else
    OBJS="$OBJS $f"
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libmugv_b200.so $OBJS -lcudart -lnccl
echo built $OUT/libmugv_b200.so
