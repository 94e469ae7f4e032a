#!/bin/bash
# Build an experiment variant of the library: flash_tc.cu (+ any other sources given in SRCS) with
# extra -D flags, linked with the production objects, into exp/<name>/libdfss_sm100a.so.
# usage: bash tools/exp_build.sh <name> "<nvcc flags>"    then  DFSS_LIB=exp/<name>/libdfss_sm100a.so python ...
NAME=$1; FLAGS=$2; SRCS=${SRCS:-flash_tc}
set -e
D=exp/$NAME; mkdir -p $D
OBJS=""
for o in paper_2203_00091_b200/lib/obj/*.o; do
  b=$(basename $o .o)
  if [[ " $SRCS " == *" $b "* ]]; then
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      --expt-relaxed-constexpr $FLAGS -c paper_2203_00091_b200/csrc/$b.cu -o $D/$b.o
    OBJS="$OBJS $D/$b.o"
  else
    OBJS="$OBJS $o"
  fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/libdfss_sm100a.so $OBJS
rm -f $D/*.o
echo built $D/libdfss_sm100a.so
