"""Where does a c2 step's time go (bring-up)?  Per-step CUDA events with and without the L2
flush, and 20 back-to-back calls between one event pair, for dfss_attention and SDPA.

    python tools/time_step_gap.py
"""
import os
import sys

import numpy as np
import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_00091_b200 as dfss  # noqa: E402

B, H, N, D = [int(x) for x in os.environ.get("SHAPE", "32,12,512,64").split(",")]
q, k, v = (torch.randn(B, H, N, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
fns = {"dfss": lambda: dfss.dfss_attention(q, k, v, "2:4", out=out),
       "sdpa": lambda: F.scaled_dot_product_attention(q, k, v)}


def per_step(fn, flush, steps=20):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for s, e in ev:
        if flush:
            flush_buf.fill_(1)
        s.record()
        fn()
        e.record()
    torch.cuda.synchronize()
    return np.median([s.elapsed_time(e) for s, e in ev]) * 1e3


def batched(fn, reps=20):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / reps


for name, fn in fns.items():
    print(f"{name}: per-step flushed {per_step(fn, True):.1f} us, per-step unflushed {per_step(fn, False):.1f} us, "
          f"back-to-back {batched(fn):.1f} us")
# graph-captured dfss step
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    fns["dfss"]()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        fns["dfss"]()
torch.cuda.current_stream().wait_stream(s)
print(f"dfss graph replay: per-step flushed {per_step(g.replay, True):.1f} us, unflushed {per_step(g.replay, False):.1f} us")
