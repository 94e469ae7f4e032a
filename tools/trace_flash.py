"""Run one c4-shaped dfss_attention with DFSS_FLASH_TRACE and print the CTA-0 pipeline timeline (bring-up).

Needs a trace build: DFSS_NVCC_EXTRA=-DDFSS_FLASH_TRACE_BUILD python -c "from paper_2203_00091_b200 import build; build.build(force=True)"
"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
out_file = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/flash_trace.bin"
if os.environ.get("DFSS_FLASH_TRACE") is None:
    import subprocess
    env = dict(os.environ, DFSS_FLASH_TRACE=out_file)
    subprocess.run([sys.executable, __file__, out_file], env=env, check=True)
    sys.exit(0)
import torch
import paper_2203_00091_b200 as dfss
shape = [int(x) for x in os.environ.get("TRACE_SHAPE", "8,12,4096,64").split(",")]
q, k, v = (torch.randn(*shape, device="cuda", dtype=torch.bfloat16) for _ in range(3))
bm = None
if os.environ.get("TRACE_MASK") == "all":  # all-kept block mask: the masked kernel on a dense pattern
    bm = dfss.BlockMask(np.ones((shape[2] // 32, shape[2] // 64), dtype=bool), 32, 64)
for _ in range(3):
    dfss.dfss_attention(q, k, v, "2:4", block_mask=bm)
torch.cuda.synchronize()
