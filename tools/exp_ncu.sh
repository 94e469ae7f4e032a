#!/bin/bash
# ncu --set full capture of the fused kernel at c4 for an exp/<variant> library
# usage: bash tools/exp_ncu.sh <variant> [tag]
V=$1; TAG=${2:-x}
mkdir -p gpurun_out
CONFIGS=c4 DFSS_LIB=exp/$V/libdfss_sm100a.so timeout -s KILL 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on \
  -k regex:dfss_flash -s 3 -c 1 -o gpurun_out/exp_${TAG}_${V} python tools/time_flash.py > gpurun_out/exp_${TAG}_${V}.log 2>&1
