#!/bin/bash
# ncu evidence for the fused flash-DFSS kernel: launch lists (c2, c4) + one --set full capture at c4.
# usage: bash tools/prof_flash.sh <tag>
TAG=${1:-r01e}
mkdir -p gpurun_out
export DFSS_BENCH_SOAK_S=0
NCU=/usr/local/cuda/bin/ncu
for CFG in c2 c4; do
timeout -s KILL 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_${TAG}_${CFG}.csv python bench.py --config $CFG --steps 2 --warmup 3 --no-extra \
   > gpurun_out/launches_${TAG}_${CFG}.log 2>&1
done
for CFG in c2 c4; do
timeout -s KILL 900 $NCU --set full --clock-control none --import-source on -k regex:dfss_flash -s 3 -c 1 \
   -o gpurun_out/prof_${TAG}_${CFG}_flash python bench.py --config $CFG --steps 1 --warmup 3 --no-extra \
   > gpurun_out/prof_${TAG}_${CFG}_flash.log 2>&1
done
echo "rc=$?"
ls -la gpurun_out/
