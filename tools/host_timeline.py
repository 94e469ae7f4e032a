"""Per-piece timeline of the dfss_attention_host pipeline at the c2 shape (bring-up): the same
three-stream schedule with timing events, printed relative to the start (ms)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_00091_b200 as dfss

q, k, v = (torch.randn((32, 12, 512, 64)).to(torch.bfloat16).pin_memory() for _ in range(3))
out = torch.empty_like(q).pin_memory()
chunks = int(sys.argv[1]) if len(sys.argv) > 1 else 4
bh, n, d = 384, 512, 64
qf, kf, vf, of = (x.view(bh, n, d) for x in (q, k, v, out))
s_in, s_run, s_out = (torch.cuda.Stream() for _ in range(3))
bounds = [bh * i // chunks for i in range(chunks + 1)]
w = bounds[1]
dq = torch.empty((2, 3, w, n, d), dtype=q.dtype, device="cuda")
do = torch.empty((2, w, n, d), dtype=q.dtype, device="cuda")
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def run():
    cur = torch.cuda.current_stream()
    start = E()
    start.record(cur)
    marks = []
    copied, ran, drained = [], [], []
    for i in range(chunks):
        lo, hi = bounds[i], bounds[i + 1]
        slot = i % 2
        with torch.cuda.stream(s_in):
            s_in.wait_event(start)
            if i >= 2:
                s_in.wait_event(ran[i - 2])
            a = E(); a.record(s_in)
            for j, src in enumerate((qf, kf, vf)):
                dq[slot, j, :hi - lo].copy_(src[lo:hi], non_blocking=True)
            copied.append(E()); copied[i].record(s_in)
        with torch.cuda.stream(s_run):
            s_run.wait_event(copied[i])
            if i >= 2:
                s_run.wait_event(drained[i - 2])
            b = E(); b.record(s_run)
            dfss.dfss_attention(dq[slot, 0], dq[slot, 1], dq[slot, 2], "2:4", out=do[slot])
            ran.append(E()); ran[i].record(s_run)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ran[i])
            c = E(); c.record(s_out)
            of[lo:hi].copy_(do[slot], non_blocking=True)
            drained.append(E()); drained[i].record(s_out)
        marks.append((a, copied[i], b, ran[i], c, drained[i]))
    cur.wait_event(drained[-1])
    return start, marks


for _ in range(3):
    run()
torch.cuda.synchronize()
start, marks = run()
torch.cuda.synchronize()
for i, m in enumerate(marks):
    print(i, " ".join(f"{start.elapsed_time(e):.3f}" for e in m), "(h2d start/end, kernel start/end, d2h start/end)")
