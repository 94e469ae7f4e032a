"""PCIe H2D / D2H bandwidth alone and concurrently (pinned buffers, separate streams)."""
import torch
n = 64 << 20
h1, h2 = torch.empty(n, dtype=torch.uint8).pin_memory(), torch.empty(n, dtype=torch.uint8).pin_memory()
d1, d2 = torch.empty(n, dtype=torch.uint8, device="cuda"), torch.empty(n, dtype=torch.uint8, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, it=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


def h2d():
    with torch.cuda.stream(sa):
        d1.copy_(h1, non_blocking=True)
    torch.cuda.current_stream().wait_stream(sa)


def d2h():
    with torch.cuda.stream(sb):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(sb)


def both():
    sa.wait_stream(torch.cuda.current_stream()); sb.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(sa):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(sb):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(sa); torch.cuda.current_stream().wait_stream(sb)


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = t(fn)
    print(f"{name}: {ms:.3f} ms  {n / ms / 1e6:.1f} GB/s per direction")
