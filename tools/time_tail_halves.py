"""n % 256 == 128 (one-set fused kernel) vs the same call through the masked two-set kernel with an
all-kept 128 x 128 BlockMask (bring-up; the masked route loses: mask preparation + masked-step
overhead)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2203_00091_b200 as dfss
def t(f, it=30):
    for _ in range(3): f()
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / it
for n in (384, 640, 896):
    q, k, v = (torch.randn(8, 12, n, 64, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    m = dfss.BlockMask(np.ones((n // 128, n // 128), dtype=bool), 128, 128)
    print(n, "unmasked", round(t(lambda: dfss.dfss_attention(q, k, v, "2:4")), 4), "all-kept mask", round(t(lambda: dfss.dfss_attention(q, k, v, "2:4", block_mask=m)), 4),
          dfss.attention_path("2:4", q.dtype, n, 64), dfss.attention_path("2:4", q.dtype, n, 64, block_mask=m))
