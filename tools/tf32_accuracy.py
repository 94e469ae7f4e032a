"""Accuracy of the fused tf32 1:2 kernel against the EXACT fp32 reference (not tf32-truncated
operands): output error statistics and the kept-mask flip rate of tf32 scores vs fp64 scores on
the same fp32 inputs (the survey asked for 5e-3 vs exact fp32 with flips counted).  Writes
profiles/tf32_accuracy.txt."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2203_00091_b200 as dfss
from oracle import oracle_c, nmattn_oracle as ref

lines = []
for n in (384, 512, 1024, 2048):
    g = torch.Generator().manual_seed(n)
    q, k, v = (torch.randn((1, 4, n, 64), generator=g) for _ in range(3))
    out = dfss.dfss_attention(q.cuda(), k.cuda(), v.cuda(), "1:2", math_mode="tf32").cpu().double().numpy()[0]
    q64, k64, v64 = (x.double().numpy()[0] for x in (q, k, v))
    want = oracle_c.attention_batched(q64, k64, v64, "1:2", nthreads=8)
    err = np.abs(out - want)
    rel = err / (np.abs(want) + 1e-3)
    # kept-mask flips: 1:2 pairs whose winner differs between tf32-truncated and exact scores
    def tf32(x):
        u = x.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)
        return u.view(np.float32).astype(np.float64)
    flips = pairs = 0
    for h in range(4):
        s_exact = q64[h] @ k64[h].T
        s_tf32 = tf32(q64[h]) @ tf32(k64[h]).T
        a = s_exact[:, 1::2] > s_exact[:, 0::2]
        b = s_tf32[:, 1::2] > s_tf32[:, 0::2]
        flips += int((a != b).sum())
        pairs += a.size
    lines.append(f"n={n} [1,4,n,64] tf32 1:2 vs exact fp32 reference: max|err| {err.max():.2e}, "
                 f"p99.9 |err| {np.quantile(err, 0.999):.2e}, mean |err| {err.mean():.2e}, "
                 f"max |err| / max|ref| {err.max() / np.abs(want).max():.2e}; kept-mask flips "
                 f"(tf32-truncated vs exact scores) {flips}/{pairs} = {flips / pairs:.2e}")
out = "\n".join(lines)
print(out)
os.makedirs("profiles", exist_ok=True)
open("profiles/tf32_accuracy.txt", "w").write(out + "\n")
