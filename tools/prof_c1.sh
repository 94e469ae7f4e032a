#!/bin/bash
# ncu evidence for the exact-FP32 c1 path: launch list + --set full of the SDDMM and the softmax-fused SpMM
TAG=${1:-r01m}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout -s KILL 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_${TAG}_c1.csv python bench.py --config c1 --steps 2 --warmup 3 --no-extra \
   > gpurun_out/launches_${TAG}_c1.log 2>&1
timeout -s KILL 600 $NCU --set full --clock-control none --import-source on -k regex:spmm_simt_softmax -s 3 -c 1 \
   -o gpurun_out/prof_${TAG}_c1_spmm python bench.py --config c1 --steps 1 --warmup 3 --no-extra \
   > gpurun_out/prof_${TAG}_c1_spmm.log 2>&1
timeout -s KILL 600 $NCU --set full --clock-control none --import-source on -k regex:sddmm_simt -s 3 -c 1 \
   -o gpurun_out/prof_${TAG}_c1_sddmm python bench.py --config c1 --steps 1 --warmup 3 --no-extra \
   > gpurun_out/prof_${TAG}_c1_sddmm.log 2>&1
echo "rc=$?"
