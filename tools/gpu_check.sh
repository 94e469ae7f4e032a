#!/bin/bash
# Bring-up run on the GPU box: probe, SIMT-path tests, then the full GPU suite.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
( timeout -s KILL 120 python tools/probe_sp.py > gpurun_out/probe.log 2>&1; echo "probe rc=$?" >> gpurun_out/probe.log )
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf --timeout 300 \
   -k "${PYTEST_K:-ffma or prune or select or meta or from_logical or softmax or c1 or golden or rel_l2 or identical or block_mask or identity or linear or single_nonzero}" \
   > gpurun_out/pytest_simt.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_simt.log
timeout -s KILL 1200 python -m pytest tests -m gpu -q -rf --timeout 300 > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
tail -5 gpurun_out/probe.log gpurun_out/pytest_simt.log gpurun_out/pytest_all.log
