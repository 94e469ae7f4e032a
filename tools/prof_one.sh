#!/bin/bash
# usage: bash tools/prof_one.sh <tag> <config> <kernel-regex>
TAG=$1; CFG=$2; K=$3
mkdir -p gpurun_out
export DFSS_BENCH_SOAK_S=0
timeout -s KILL 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
   -o gpurun_out/prof_${TAG}_${CFG}_${K} python bench.py --config $CFG --steps 1 --warmup 3 --no-extra \
   > gpurun_out/prof_${TAG}_${CFG}_${K}.log 2>&1
echo "rc=$?"
