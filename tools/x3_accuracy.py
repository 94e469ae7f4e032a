"""3xTF32 score accuracy, emulated on the CPU (numpy): scores of the c1 inputs (and 8 heads at
n = 1024) from Qh Kh^T + Qh Kl^T + Ql Kh^T with round-to-nearest tf32 splits, against float64,
next to the plain fp32 product -- maximum error and 1:2 selection flips (pair winner differs
from the float64 one).  Backs the exact-FP32 3xTF32 path (csrc/sddmm_tf32.cu).

    python tools/x3_accuracy.py
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch


def tf32(x):  # round to nearest (ties away) at a 10-bit mantissa, as cvt.rna.tf32.f32
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    return (((u + 0x1000) & 0xFFFFE000).astype(np.uint32)).view(np.float32)


def compare(shape, seed):
    g = torch.Generator().manual_seed(seed)
    q, k = [torch.randn(shape, generator=g, dtype=torch.float32).numpy().reshape(-1, shape[-2], shape[-1])
            for _ in range(2)]
    flips32 = flipsx3 = 0
    err32 = errx3 = 0.0
    for a, b in zip(q, k):
        s64 = (a.astype(np.float64) @ b.T.astype(np.float64)) / 8
        s32 = (a @ b.T).astype(np.float32) / np.float32(8)
        ah, bh = tf32(a), tf32(b)
        al, bl = tf32(a - ah), tf32(b - bh)
        sx3 = ((ah @ bl.T).astype(np.float32) + (al @ bh.T).astype(np.float32) + (ah @ bh.T).astype(np.float32)) / np.float32(8)
        win = lambda s: s[:, 1::2] > s[:, 0::2]  # noqa: E731
        flips32 += int((win(s32) != win(s64)).sum())
        flipsx3 += int((win(sx3) != win(s64)).sum())
        err32 = max(err32, float(np.abs(s32 - s64).max()))
        errx3 = max(errx3, float(np.abs(sx3 - s64).max()))
    print(f"{shape}: max |err| fp32 {err32:.3e}  3xtf32 {errx3:.3e};  1:2 flips vs float64: fp32 {flips32}  3xtf32 {flipsx3}")


compare((1, 12, 384, 64), 0)
compare((1, 8, 1024, 64), 5)
