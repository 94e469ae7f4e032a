"""Time the flash kernel under DFSS_FLASH_DEBUG variants (bring-up experiment; each variant in a fresh process)."""
import os, subprocess, sys, json
code = r'''
import torch, sys
sys.path.insert(0, ".")
import paper_2203_00091_b200 as dfss
n = int(sys.argv[1]); bh = int(sys.argv[2])
q, k, v = (torch.randn(bh, n, 64, device="cuda", dtype=torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
ws = torch.empty(dfss.workspace_bytes("2:4", q.dtype, bh, n, 64), dtype=torch.uint8, device="cuda")
for _ in range(3): dfss.dfss_attention(q, k, v, "2:4", out=out, workspace=ws)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): dfss.dfss_attention(q, k, v, "2:4", out=out, workspace=ws)
e.record(); torch.cuda.synchronize()
print(s.elapsed_time(e) / 10)
'''
res = {}
for n, bh in ((4096, 96),):
    for dbg in [int(x) for x in os.environ.get('VARIANTS', '0,1,4,5,7,15,23,31,13').split(',')]:
        env = dict(os.environ, DFSS_FLASH_DEBUG=str(dbg))
        out = subprocess.run([sys.executable, "-c", code, str(n), str(bh)], env=env, capture_output=True, text=True)
        res[f"n{n}_dbg{dbg}"] = out.stdout.strip() or out.stderr.strip()[-200:]
        print(n, dbg, res[f"n{n}_dbg{dbg}"], flush=True)
