"""Does tcgen05.mma ever produce -0 scores?  Runs the staged SDDMM with a raw-score dump on inputs built to
produce exact-zero dot products from signed zeros, and counts -0.0 in the fp32 score dump (bring-up check)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_00091_b200 as dfss

n, d = 256, 64
cases = {}
z = torch.zeros((1, 1, n, d))
pos = torch.rand((1, 1, n, d)) + 0.5
for name, (q, k) in {"q=+0,k>0": (z, pos), "q=-0,k>0": (-z, pos), "q=+0,k<0": (z, -pos), "q=-0,k<0": (-z, -pos),
                     "q=mixed0,k=+-": (torch.where(torch.rand_like(z) < .5, z, -z), torch.where(torch.rand_like(pos) < .5, pos, -pos))}.items():
    qb, kb = q.to(torch.bfloat16).cuda(), k.to(torch.bfloat16).cuda()
    dbg = torch.empty((1, 1, n, n), dtype=torch.float32, device="cuda")
    dfss.sddmm_prune(qb, kb, "2:4", 1.0, scores_out=dbg)  # scale 1.0: fma(s, 1, +0) canonicalizes, so also dump raw
    raw = torch.empty_like(dbg)
    torch.cuda.synchronize()
    neg = int((dbg.view(torch.int32) == -2**31).sum())
    cases[name] = neg
print(cases)
