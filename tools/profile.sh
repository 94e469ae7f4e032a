#!/bin/bash
# ncu evidence for profiles/: launch list (share of the step) + one full capture per hot kernel.
# usage: bash tools/profile.sh <tag> [config]
TAG=${1:-r01}; CFG=${2:-c2}
mkdir -p gpurun_out
export DFSS_BENCH_SOAK_S=0
NCU=/usr/local/cuda/bin/ncu
timeout -s KILL 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_${TAG}_${CFG}.csv python bench.py --config $CFG --steps 2 --warmup 3 --no-extra \
   > gpurun_out/launches_${TAG}_${CFG}.log 2>&1
# full sets: skip the warm-up launches of each kernel (-s), capture one timed launch each
for K in sddmm24_tc softmax_rows spmm24_tc; do
  timeout -s KILL 900 $NCU --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
     -o gpurun_out/prof_${TAG}_${CFG}_${K} python bench.py --config $CFG --steps 1 --warmup 3 --no-extra \
     > gpurun_out/prof_${TAG}_${CFG}_${K}.log 2>&1
done
ls -la gpurun_out/
