#!/bin/bash
# Quick GPU pass (bring-up): full -m gpu suite, then ncu launch lists of the fused kernel at c2 / c4.
# usage: bash tools/gpu_quick.sh [tag]
TAG=${1:-q}
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}.log
for C in ${CONFIGS:-c2 c4}; do
  timeout -s KILL 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}_${C}.csv python bench.py --config $C --steps 2 --warmup 3 --no-extra > /dev/null 2>&1
done
tail -2 gpurun_out/pytest_${TAG}.log
