"""Staged (reference-shaped) kernels at c4 / c2: sddmm_prune, softmax_rows, spmm -- per-kernel time
and the fraction of the measured HBM copy bandwidth their algorithmic bytes imply (bring-up)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_00091_b200 as dfss

HBM = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json"))).get("hbm_gbs", 6548.0) if os.path.exists("MEASURED_PEAKS.json") else 6548.0


def t_ms(fn, it=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it


for name, (b, h, n, dt, mode) in {"c2": (32, 12, 512, torch.bfloat16, "2:4"), "c4": (8, 12, 4096, torch.bfloat16, "2:4"),
                                  "c4_12": (8, 12, 4096, torch.bfloat16, "1:2"),
                                  "c3": (16, 16, 1024, torch.float16, "2:4"), "c4h": (8, 12, 4096, torch.float16, "2:4")}.items():
    if os.environ.get("CONFIGS") and name not in os.environ["CONFIGS"].split(","):
        continue
    q, k, v = (torch.randn(b, h, n, 64, device="cuda", dtype=dt) for _ in range(3))
    bh = b * h
    c, _ = dfss.attention_sddmm(q, k, mode)
    nzb = c.nonzeros.numel() * c.nonzeros.element_size()
    metab = c.meta_hw.numel() * 4
    ts = t_ms(lambda: dfss.attention_sddmm(q, k, mode))
    tsm = t_ms(lambda: dfss.softmax_rows(c, check=False))
    p = dfss.softmax_rows(c, check=False)
    tp = t_ms(lambda: dfss.spmm(p, v))
    qkv = bh * n * 64 * 2
    for kname, ms, nbytes in (("sddmm_prune", ts, nzb + metab + 2 * qkv), ("softmax_rows", tsm, 2 * nzb),
                              ("spmm", tp, nzb + metab + 2 * qkv)):
        print(f"{name} {mode} {kname:13s} {ms:.4f} ms  {nbytes / ms / 1e6:.0f} GB/s = {nbytes / ms / 1e6 / HBM:.2f} of HBM", flush=True)
