#!/bin/bash
# Iteration pass on the GPU box: timing vs SDPA (c2, c3, c4), then the GPU suite.
# usage: bash tools/gpu_iter.sh [tag] [pytest -k expression]
TAG=${1:-it}
mkdir -p gpurun_out
timeout -s KILL 300 python tools/time_flash.py > gpurun_out/time_${TAG}.log 2>&1
DFSS_MODE=1:2 timeout -s KILL 300 python tools/time_flash.py >> gpurun_out/time_${TAG}.log 2>&1
if [ -n "$2" ]; then K="-k $2"; else K=""; fi
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x --timeout 300 $K > gpurun_out/pytest_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}.log
cat gpurun_out/time_${TAG}.log; tail -3 gpurun_out/pytest_${TAG}.log
