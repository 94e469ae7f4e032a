"""dfss_attention_host timing vs raw copies (c2 shape)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_00091_b200 as dfss

q, k, v = (torch.randn((32, 12, 512, 64)).to(torch.bfloat16).pin_memory() for _ in range(3))
out = torch.empty_like(q).pin_memory()


def t(fn, it=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


for c in (1, 2, 4, 8, 16):
    print("chunks", c, round(t(lambda: dfss.dfss_attention_host(q, k, v, "2:4", out=out, chunks=c)), 3), "ms")
dq = torch.empty((3,) + q.shape, dtype=q.dtype, device="cuda")
print("raw h2d", round(t(lambda: [dq[i].copy_(x, non_blocking=True) for i, x in enumerate((q, k, v))]), 3))
print("raw d2h", round(t(lambda: out.copy_(dq[0], non_blocking=True)), 3))
