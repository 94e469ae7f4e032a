"""c1 (1:2 fp32 exact, [1,12,384,64]) staged-path timing (kernel view)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_00091_b200 as dfss
q, k, v = (torch.randn(1, 12, 384, 64, device="cuda") for _ in range(3))
out = torch.empty_like(q)
ws = torch.empty(dfss.workspace_bytes("1:2", torch.float32, 12, 384, 64, "ffma"), dtype=torch.uint8, device="cuda")
f = lambda: dfss.dfss_attention(q, k, v, "1:2", math_mode="ffma", out=out, workspace=ws)  # noqa: E731
for _ in range(5):
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    f()
e1.record()
torch.cuda.synchronize()
print("c1 exact fp32:", round(e0.elapsed_time(e1) / 50, 4), "ms")
