"""Host cost per call of dfss_attention vs torch SDPA (bring-up): many calls on a tiny shape
whose kernel is a few microseconds, so the wall time per call is the host path.

    python tools/time_call_overhead.py
"""
import os
import sys
import time

import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_00091_b200 as dfss  # noqa: E402

q, k, v = (torch.randn(1, 1, 256, 64, device="cuda", dtype=torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
ws = torch.empty(max(dfss.workspace_bytes("2:4", q.dtype, 1, 256, 64), 1), dtype=torch.uint8, device="cuda")
for name, fn in [("dfss_attention", lambda: dfss.dfss_attention(q, k, v, "2:4", out=out, workspace=ws)),
                 ("sdpa", lambda: F.scaled_dot_product_attention(q, k, v))]:
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2000):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name}: host {1e6 * (t1 - t0) / 2000:.2f} us/call, wall {1e6 * (t2 - t0) / 2000:.2f} us/call")
