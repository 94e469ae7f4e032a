#!/bin/bash
# build libdfss variants with DFSS_MASK_EXP=<bits> into paper_2203_00091_b200/lib/exp/ (CPU side)
set -e
cd "$(dirname "$0")/.."
O=paper_2203_00091_b200/lib/obj
mkdir -p paper_2203_00091_b200/lib/exp
for e in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -DDFSS_MASK_EXP=$e -c paper_2203_00091_b200/csrc/flash_tc.cu -o /tmp/flash_exp_$e.o
  objs=$(ls $O/*.o | grep -v flash_tc.o)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2203_00091_b200/lib/exp/lib_$e.so /tmp/flash_exp_$e.o $objs
done
