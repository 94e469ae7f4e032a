"""Fused 2:4 bf16 over the configs[4] sequence lengths (batch 8 x 12 heads) and c2 / c4, unflushed (bring-up)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_00091_b200 as dfss

for b, h, n in ((8, 12, 384), (8, 12, 512), (8, 12, 768), (8, 12, 1024), (8, 12, 2048), (32, 12, 512), (8, 12, 4096)):
    q, k, v = (torch.randn(b, h, n, 64, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    f = lambda: dfss.dfss_attention(q, k, v, "2:4")  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"[{b},{h},{n}] {e0.elapsed_time(e1) / 20:.4f} ms", flush=True)
