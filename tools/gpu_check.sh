#!/bin/bash
# Bring-up run on the GPU box: probe, full GPU suite, then a bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
( timeout -s KILL 120 python tools/probe_sp.py > gpurun_out/probe.log 2>&1; echo "probe rc=$?" >> gpurun_out/probe.log )
timeout -s KILL 1200 python -m pytest tests -m gpu -q -rf --timeout 300 ${PYTEST_ARGS} > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
if [ -z "$NO_BENCH" ]; then
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
fi
tail -3 gpurun_out/probe.log gpurun_out/pytest_all.log gpurun_out/bench.err
