"""Shared helpers for the GPU parity tests (inputs, oracle comparison)."""

from __future__ import annotations

import numpy as np
import torch

from oracle import nmattn_oracle as ref
from oracle import oracle_c


def seeded_qkv(shape, dtype, seed=0, scale=1.0):
    """draw N(0,1) in fp32 with a torch Generator, cast to the run
    dtype on the host, copy to the GPU; the oracle gets float64 of the rounded values."""
    g = torch.Generator().manual_seed(seed)
    out = []
    for _ in range(3):
        x = (torch.randn(shape, generator=g, dtype=torch.float32) * scale).to(dtype)
        out.append(x)
    return [x.cuda() for x in out], [x.double().numpy() for x in out]


def logical_meta(c) -> np.ndarray:
    """[..., rows, groups] uint8 logical nibbles of a GPU CompressedSparse."""
    return c.meta_grid().cpu().numpy()


def oracle_on_scores(scores: np.ndarray, mode: str):
    """compress_logical + prune_dense of the reference on the given scores (codec.py:324-335)."""
    kept, nz, nib = ref.select_rows(scores, mode)
    return nz, nib, kept


def assert_close(got, want, rtol, atol, what=""):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    err = np.abs(got - want)
    bound = atol + rtol * np.abs(want)
    bad = err > bound
    if bad.any():
        idx = np.unravel_index(np.argmax(err - bound), err.shape)
        raise AssertionError(
            f"{what}: {int(bad.sum())} / {bad.size} elements outside |d| <= {atol} + {rtol}|ref|; "
            f"worst at {idx}: got {got[idx]!r} want {want[idx]!r}"
        )


def oracle_attention(q64, k64, v64, mode):
    """Reference nm_attention per (batch, head) via the C restatement (bitwise = numba)."""
    shp = q64.shape
    n, d = shp[-2], shp[-1]
    flat = lambda x: x.reshape(-1, n, d)
    out = oracle_c.attention_batched(flat(q64), flat(k64), flat(v64), mode, nthreads=8)
    return out.reshape(shp)
