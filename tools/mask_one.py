"""One unmasked and one all-kept-masked fused call (for ncu launch lists)."""
import numpy as np, torch
import paper_2203_00091_b200 as dfss
n, bh = 4096, 64
q, k, v = [torch.randn((1, bh, n, 64), device="cuda").to(torch.bfloat16) for _ in range(3)]
bm = dfss.BlockMask(np.ones((n // 32, n // 64), bool), 32, 64)
for _ in range(2):
    dfss.dfss_attention(q, k, v, "2:4")
    dfss.dfss_attention(q, k, v, "2:4", block_mask=bm)
torch.cuda.synchronize()
