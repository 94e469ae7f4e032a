"""Why the first L2-flushed step after warm-up is slow (bring-up): per-step times under three
warm-up patterns, DFSS and SDPA, c2."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_00091_b200 as dfss

q, k, v = (torch.randn(384, 512, 64, device="cuda", dtype=torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
buf = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
fns = {"dfss": lambda: dfss.dfss_attention(q, k, v, "2:4", out=out),
       "sdpa": lambda: torch.nn.functional.scaled_dot_product_attention(q[None], k[None], v[None])}
for name, fn in fns.items():
    for pat in ("warm-unflushed+sync", "warm-flushed+sync", "warm-flushed-nosync", "two-flushes+sync"):
        for _ in range(3):
            if pat != "warm-unflushed+sync":
                buf.fill_(1)
            fn()
        if "nosync" not in pat:
            torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(8)]
        for s, e in ev:
            buf.fill_(1)
            if pat == "two-flushes+sync":
                buf.fill_(2)
            s.record(); fn(); e.record()
        torch.cuda.synchronize()
        print(f"{name} {pat:22s}: " + " ".join(f"{s.elapsed_time(e):.4f}" for s, e in ev), flush=True)
