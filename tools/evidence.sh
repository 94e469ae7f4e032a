#!/bin/bash
# One GPU evidence pass: GPU suite, smoke, bench line, ncu launch lists (c2, c4) + one --set full capture of the fused kernel.
# usage: bash tools/evidence.sh <tag> [skip-tests]
TAG=${1:-r02a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_${TAG}.txt 2>&1
if [ -z "$2" ]; then
timeout -s KILL 1500 python -m pytest tests -m gpu -q -rf --timeout 300 > gpurun_out/pytest_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_${TAG}.log
fi
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?" >> gpurun_out/bench_${TAG}.err
bash tools/prof_flash.sh ${TAG} > /dev/null 2>&1
tail -n 3 gpurun_out/pytest_${TAG}.log gpurun_out/smoke_${TAG}.log gpurun_out/bench_${TAG}.err
