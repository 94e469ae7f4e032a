"""Exact-FP32 1:2 attention (staged SIMT path) over the configs[4] sequence lengths, batch 8 x 12 heads."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_00091_b200 as dfss
for n in (384, 512, 768, 1024):
    q, k, v = (torch.randn(8, 12, n, 64, device="cuda") for _ in range(3))
    out = torch.empty_like(q)
    ws = torch.empty(dfss.workspace_bytes("1:2", torch.float32, 96, n, 64, os.environ.get("MATH", "auto")), dtype=torch.uint8, device="cuda")
    f = lambda: dfss.dfss_attention(q, k, v, "1:2", math_mode=os.environ.get("MATH", "auto"), out=out, workspace=ws)  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"n={n}: {e0.elapsed_time(e1) / 10:.4f} ms", flush=True)
