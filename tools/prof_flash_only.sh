#!/bin/bash
# one --set full capture of the fused kernel at a config: bash tools/prof_flash_only.sh <tag> <cfg>
TAG=${1:-x}; CFG=${2:-c4}
mkdir -p gpurun_out
export DFSS_BENCH_SOAK_S=0
timeout -s KILL 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:dfss_flash -s 3 -c 1 \
   -o gpurun_out/prof_${TAG}_${CFG}_flash python bench.py --config $CFG --steps 1 --warmup 3 --no-extra \
   > gpurun_out/prof_${TAG}_${CFG}_flash.log 2>&1
echo "rc=$?"
