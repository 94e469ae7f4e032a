"""Time the fused kernel with no mask, an all-kept mask, and block-causal masks."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2203_00091_b200 as dfss

n, bh = 4096, 64
g = torch.Generator().manual_seed(3)
q, k, v = [torch.randn((1, bh, n, 64), generator=g).to(torch.bfloat16).cuda() for _ in range(3)]
out = torch.empty_like(q)


def causal(tr, tc_, blk):
    rows = np.arange(n // tr) * tr // blk
    cols = np.arange(n // tc_) * tc_ // blk
    return dfss.BlockMask(cols[None, :] <= rows[:, None], tr, tc_)


def timed(bm, mode="2:4"):
    for _ in range(3):
        dfss.dfss_attention(q, k, v, mode, block_mask=bm, out=out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        dfss.dfss_attention(q, k, v, mode, block_mask=bm, out=out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 10


for mode in ("2:4", "1:2"):
    print(mode, "none", timed(None, mode))
    print(mode, "all-kept", timed(dfss.BlockMask(np.ones((n // 32, n // 64), bool), 32, 64), mode))
    print(mode, "causal128", timed(causal(32, 64, 128), mode))
    print(mode, "causal256", timed(causal(32, 64, 256), mode))
    print(mode, "causal32", timed(causal(32, 64, 32), mode))

q, k, v = (x.float() for x in (q, k, v))
out = torch.empty_like(q)


def timed32(bm):
    f = lambda: dfss.dfss_attention(q, k, v, "1:2", math_mode="tf32", block_mask=bm, out=out)  # noqa: E731
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 10


print("tf32 1:2 none", timed32(None))
print("tf32 1:2 all-kept", timed32(dfss.BlockMask(np.ones((n // 32, n // 64), bool), 32, 64)))
print("tf32 1:2 causal128", timed32(causal(32, 64, 128)))
