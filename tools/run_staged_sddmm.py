"""Run the staged tcgen05 SDDMM a few times at the c4 shape (ncu target; bring-up)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_00091_b200 as dfss

mode = os.environ.get("MODE", "2:4")
q, k = (torch.randn(8, 12, 4096, 64, device="cuda", dtype=torch.bfloat16) for _ in range(2))
for _ in range(4):
    dfss.attention_sddmm(q, k, mode)
torch.cuda.synchronize()
