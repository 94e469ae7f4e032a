"""Quick timing of dfss_attention vs SDPA at the bench configs (bring-up; bench.py is the contract)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_00091_b200 as dfss

def t_ms(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it

import os as _os
MODE = _os.environ.get("DFSS_MODE", "2:4")
for name, (b, h, n, dt) in {"c2": (32, 12, 512, torch.bfloat16), "c3": (16, 16, 1024, torch.float16),
                             "c4": (8, 12, 4096, torch.bfloat16)}.items():
    if _os.environ.get("CONFIGS") and name not in _os.environ["CONFIGS"].split(","):
        continue
    q, k, v = (torch.randn(b, h, n, 64, device="cuda", dtype=dt) for _ in range(3))
    out = torch.empty_like(q)
    ws = torch.empty(dfss.workspace_bytes(MODE, dt, b * h, n, 64), dtype=torch.uint8, device="cuda")
    a = t_ms(lambda: dfss.dfss_attention(q, k, v, MODE, out=out, workspace=ws))
    s = t_ms(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v))
    print(f"{name} {MODE}: dfss {a:.4f} ms  sdpa {s:.4f} ms  speedup {s / a:.3f}x", flush=True)
