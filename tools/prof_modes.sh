#!/bin/bash
# ncu --set full captures of the fused kernels in each mode at the c4 shape [8,12,4096,64]
TAG=${1:-r01h}
mkdir -p gpurun_out
cat > /tmp/run_mode.py <<'PY'
import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2203_00091_b200 as dfss
mode, dt, mm = sys.argv[1], {"bf16": torch.bfloat16, "f32": torch.float32}[sys.argv[2]], sys.argv[3]
q, k, v = (torch.randn(8, 12, 4096, 64, device="cuda", dtype=dt) for _ in range(3))
for _ in range(3):
    dfss.dfss_attention(q, k, v, mode, math_mode=mm)
torch.cuda.synchronize()
PY
for spec in "1:2 bf16 auto 12" "1:2 f32 tf32 tf32" "2:4 bf16 auto 24"; do
  set -- $spec
  timeout -s KILL 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:dfss_flash -s 2 -c 1 \
     -o gpurun_out/prof_${TAG}_c4_flash$4 python /tmp/run_mode.py $1 $2 $3 > gpurun_out/prof_${TAG}_$4.log 2>&1
done
ls gpurun_out | grep ${TAG}
