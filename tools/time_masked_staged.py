"""Masked staged (reference-shaped) path at the c4 shape: sddmm_prune / softmax_rows / spmm with a
block-causal BlockMask on 32 x 64 tiles (bring-up timing)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2203_00091_b200 as dfss

def t_ms(fn, it=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it

b, h, n = 8, 12, 4096
q, k, v = (torch.randn(b, h, n, 64, device="cuda", dtype=torch.bfloat16) for _ in range(3))
rows, cols = np.arange(n // 32) * 32 // 128, np.arange(n // 64) * 64 // 128
mask = dfss.BlockMask(cols[None, :] <= rows[:, None], 32, 64)
for mode in ("2:4", "1:2"):
    c, _ = dfss.sddmm_prune(q, k, mode, 0.125, mask)
    p = dfss.softmax_rows(c, check=False)
    print(mode, "masked sddmm_prune", round(t_ms(lambda: dfss.sddmm_prune(q, k, mode, 0.125, mask)), 3), "ms",
          "softmax", round(t_ms(lambda: dfss.softmax_rows(c, check=False)), 3), "ms",
          "spmm", round(t_ms(lambda: dfss.spmm(p, v)), 3), "ms", flush=True)
