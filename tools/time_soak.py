"""Effect of a sustained-load soak on the flushed step time (bring-up: bench.py soaks 1.5 s before timing)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import pynvml
import torch
import paper_2203_00091_b200 as dfss

pynvml.nvmlInit()
hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
flush_buf = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
SHAPE = tuple(int(x) for x in os.environ.get("SOAK_SHAPE", "8,12,4096,64").split(","))
q, k, v = (torch.randn(*SHAPE, device="cuda", dtype=torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
fns = {"dfss": lambda: dfss.dfss_attention(q, k, v, "2:4", out=out),
       "sdpa": lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v)}


def timed(fn):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    for s, e in ev:
        flush_buf.fill_(1); s.record(); fn(); e.record()
    torch.cuda.synchronize()
    return np.array([s.elapsed_time(e) for s, e in ev])


def clocks():
    return (pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(hnd) / 1000,
            pynvml.nvmlDeviceGetTemperature(hnd, pynvml.NVML_TEMPERATURE_GPU),
            hex(pynvml.nvmlDeviceGetCurrentClocksEventReasons(hnd)))


for name, fn in fns.items():
    for soak in (0.0, 1.5, 5.0):
        time.sleep(2.0)
        for _ in range(3): fn()
        torch.cuda.synchronize()
        t_end = time.perf_counter() + soak
        cl = None
        while time.perf_counter() < t_end:
            for _ in range(20): fn()
            torch.cuda.synchronize()
            cl = clocks()
        r = timed(fn)
        print(f"{name} soak {soak:.1f}s: mean {r.mean():.4f} ms  first {r[0]:.4f}  last {r[-1]:.4f}  clocks(sm MHz, W, C, reasons) during soak {cl} after {clocks()}", flush=True)
