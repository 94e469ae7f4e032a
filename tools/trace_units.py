"""Per-CTA unit timeline of the two-set kernel (trace build, bring-up): when each CTA's units
start / see their first S / finish, to see the last round (split or not).

    DFSS_NVCC_EXTRA=-DDFSS_FLASH_TRACE_BUILD python -c "from paper_2203_00091_b200 import build; build.build(force=True)"
    TRACE_SHAPE=32,12,512,64 python tools/trace_units.py gpurun_out/units.bin
"""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
out_file = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/units.bin"
if os.environ.get("DFSS_FLASH_TRACE") is None:
    subprocess.run([sys.executable, __file__, out_file], env=dict(os.environ, DFSS_FLASH_TRACE=out_file), check=True)
    raw = np.fromfile(out_file, dtype=np.uint64).astype(np.int64)
    u = raw[16 * 2 * 64 * 2:].reshape(148, 16, 8)
    base = u[u > 0].min()
    u = np.where(u > 0, u - base, -1)
    for b in list(range(0, 6)) + list(range(100, 116)) + [140, 147]:
        ks = [k for k in range(15) if u[b, k, 0] >= 0]
        print(f"cta {b:3d}: " + " | ".join(f"u{k} start {u[b, k, 0]:7d} q {u[b, k, 1]:7d} s0 {u[b, k, 2]:7d} end {u[b, k, 3]:7d}"
                                          for k in ks[-3:]) + f" | final epi {u[b, 15, 4]:7d} -> {u[b, 15, 5]:7d}")
    ends = u[:, 15, 5]
    print("kernel end (max over CTAs):", ends.max(), " median CTA end:", int(np.median(ends)))
    sys.exit(0)
import torch  # noqa: E402

import paper_2203_00091_b200 as dfss  # noqa: E402

shape = [int(x) for x in os.environ.get("TRACE_SHAPE", "32,12,512,64").split(",")]
q, k, v = (torch.randn(*shape, device="cuda", dtype=torch.bfloat16) for _ in range(3))
for _ in range(3):
    dfss.dfss_attention(q, k, v, "2:4")
torch.cuda.synchronize()
