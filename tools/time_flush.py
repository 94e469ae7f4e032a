"""Flushed vs unflushed step time of dfss_attention and SDPA at c2 / c4 (bring-up: where the bench's
L2-flushed numbers differ from back-to-back timing)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2203_00091_b200 as dfss

flush_buf = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
spin = torch.empty(64 * 2**20, dtype=torch.uint8, device="cuda")


def per_step(fn, steps=10, mode="flush"):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for s, e in ev:
        if mode in ("flush", "flush+gap"):
            flush_buf.fill_(1)
        if mode == "flush+gap":
            for _ in range(4):
                spin.fill_(2)  # small kernels after the flush: HBM-write drain / clocks settle
        s.record()
        fn()
        e.record()
    torch.cuda.synchronize()
    return float(np.median([s.elapsed_time(e) for s, e in ev]))


for name, (b, h, n, dt) in {"c2": (32, 12, 512, torch.bfloat16), "c4": (8, 12, 4096, torch.bfloat16)}.items():
    q, k, v = (torch.randn(b, h, n, 64, device="cuda", dtype=dt) for _ in range(3))
    out = torch.empty_like(q)
    f_d = lambda: dfss.dfss_attention(q, k, v, "2:4", out=out)  # noqa: E731
    f_s = lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v)  # noqa: E731
    for mode in ("none", "flush", "flush+gap"):
        print(f"{name} {mode:10s} dfss {per_step(f_d, mode=mode):.4f} ms  sdpa {per_step(f_s, mode=mode):.4f} ms", flush=True)

# clock sampling during timing: nvidia-smi spawned every 0.1 s (bench before r02) vs one -lms 200 process
import subprocess, threading, time
q, k, v = (torch.randn(8, 12, 4096, 64, device="cuda", dtype=torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
f_d = lambda: dfss.dfss_attention(q, k, v, "2:4", out=out)  # noqa: E731
Q = "clocks.sm,clocks.max.sm,power.draw"
stop = threading.Event()
def spawner():
    while not stop.is_set():
        subprocess.run(["nvidia-smi", "-i", "0", f"--query-gpu={Q}", "--format=csv,noheader"], capture_output=True)
        stop.wait(0.1)
for label in ("no sampler", "spawn every 0.1 s", "one -lms 200"):
    stop.clear()
    th = p = None
    if label.startswith("spawn"):
        th = threading.Thread(target=spawner, daemon=True); th.start()
    elif label.startswith("one"):
        p = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={Q}", "--format=csv,noheader", "-lms", "200"],
                             stdout=subprocess.DEVNULL)
    time.sleep(0.5)
    res = []
    for _ in range(20):
        for _ in range(3): f_d()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        for s, e in ev:
            flush_buf.fill_(1); s.record(); f_d(); e.record()
        torch.cuda.synchronize()
        res += [s.elapsed_time(e) for s, e in ev]
    stop.set()
    if th: th.join()
    if p: p.terminate(); p.wait()
    r = np.array(res)
    print(f"c4 flushed, {label:18s}: mean {r.mean():.4f}  median {np.median(r):.4f}  max {r.max():.4f}  >0.55ms: {(r > 0.55).sum()}/{len(r)}", flush=True)
