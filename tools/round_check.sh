#!/bin/bash
# Full GPU evidence pass: isolated GPU tests (hang-safe), smoke, bench line, ncu launch lists + one full capture.
TAG=${1:-r01f}
mkdir -p gpurun_out
T=60 bash tools/gpu_tests_isolated.sh "" > gpurun_out/tests_${TAG}.log 2>&1
grep -c "rc=0" gpurun_out/tests_${TAG}.log > gpurun_out/tests_${TAG}.summary; grep -v "rc=0" gpurun_out/tests_${TAG}.log >> gpurun_out/tests_${TAG}.summary
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_${TAG}.log
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
bash tools/prof_flash.sh ${TAG} > /dev/null 2>&1
ls gpurun_out
