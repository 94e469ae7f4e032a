"""Exact-fp32 1:2 attention, math auto vs ffma, over small (batch x heads, n) shapes (bring-up:
calibrates where the 3xTF32 tcgen05 path starts to pay)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_00091_b200 as dfss

for bh, n in ((12, 384), (24, 384), (48, 384), (12, 512), (24, 512), (12, 768), (12, 1024), (96, 384)):
    q, k, v = (torch.randn(1, bh, n, 64, device="cuda") for _ in range(3))
    res = []
    for mm in ("auto", "ffma"):
        ws = torch.empty(dfss.workspace_bytes("1:2", torch.float32, bh, n, 64, mm), dtype=torch.uint8, device="cuda")
        out = torch.empty_like(q)
        f = lambda: dfss.dfss_attention(q, k, v, "1:2", math_mode=mm, out=out, workspace=ws)  # noqa: E731
        for _ in range(5):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(30):
            f()
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / 30)
    print(f"bh={bh} n={n} scores={bh * n * n / 1e6:.1f}M  auto {res[0]:.4f} ms  ffma {res[1]:.4f} ms", flush=True)
