"""The reference's kernel module on the device, in float64 (include/dfss.h dfss_kmod_*).

The reference computes everything in float64 through five kernel functions
(``_kernels_numba.py:39,62,87,106,188``).  These are the same five on CUDA float64 tensors,
with the reference's arithmetic (one accumulator per output, ascending reduction index,
separately rounded products and sums): sddmm_compress, spmm_gather, gemm_abt and the
selection are bitwise the reference's; the softmaxes differ only through exp (<= 1 ulp).
The package routes float64 data here (DenseMatrix keeps float64; compress_logical,
prune_dense, sddmm_prune, softmax_rows, spmm, gemm_scaled, full_attention and nm_attention
dispatch on the dtype), so a float64 caller gets the reference's numbers, not an fp32
approximation.  The fused 16/32-bit kernels are the fast path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

_INT32_MAX = 2**31 - 1


def _f64(t: torch.Tensor, name: str) -> torch.Tensor:
    if t.dtype != torch.float64:
        raise ValueError(f"{name} must be float64, got {t.dtype}")
    _lib.require_cuda(t)
    return t.contiguous()


def sddmm_compress(q: torch.Tensor, k: torch.Tensor, scale: float, group_size: int, tile_rows: int, tile_cols: int,
                   keep: np.ndarray | None = None):
    """Fused score -> prune -> compress of one [n, d] x [m, d] pair (_kernels_numba.py:110-188).
    Returns (nonzeros f64 [n, m/2], logical meta uint8 [n, m/gs]); masked tiles stay zero."""
    q, k = _f64(q, "q"), _f64(k, "k")
    n, d = q.shape
    m = k.shape[0]
    if keep is None:
        keep = np.ones((-(-n // tile_rows), -(-m // tile_cols)), dtype=bool)
    dkeep = torch.from_numpy(np.ascontiguousarray(keep, dtype=np.uint8)).to(q.device)
    nz = torch.empty((n, m // 2), dtype=torch.float64, device=q.device)
    meta = torch.empty((n, m // group_size), dtype=torch.uint8, device=q.device)
    with torch.cuda.device(q.device):
        _lib.check(_lib.load().dfss_kmod_sddmm_compress(_lib.ptr(q), _lib.ptr(k), float(scale), int(group_size), n, m, d,
                                                        int(tile_rows), int(tile_cols), _lib.ptr(dkeep), _lib.ptr(nz),
                                                        _lib.ptr(meta), _lib.stream_of(q)), "sddmm_compress")
    return nz, meta


def prune_scores(scores: torch.Tensor, group_size: int, want_kept: bool = True):
    """Selection on given float64 scores [..., cols] (codec.py:289-313):
    (nonzeros f64 [..., cols/2], meta uint8 [..., cols/gs], kept uint8 [..., cols] or None)."""
    s = _f64(scores, "scores")
    cols = s.shape[-1]
    rows = s.numel() // cols if cols else 0
    nz = torch.empty(s.shape[:-1] + (cols // 2,), dtype=torch.float64, device=s.device)
    meta = torch.empty(s.shape[:-1] + (cols // group_size,), dtype=torch.uint8, device=s.device)
    kept = torch.empty(s.shape, dtype=torch.uint8, device=s.device) if want_kept else None
    with torch.cuda.device(s.device):
        _lib.check(_lib.load().dfss_prune_scores_f64(_lib.ptr(s), _lib.ptr(nz), _lib.ptr(meta), _lib.ptr(kept),
                                                     int(group_size), rows, cols, _lib.stream_of(s)), "prune_scores_f64")
    return nz, meta, kept


def softmax_nonzeros(nz: torch.Tensor, present: torch.Tensor | None = None) -> torch.Tensor:
    """Per-row softmax over present entries of [..., cols] (_kernels_numba.py:66-87); absent -> 0."""
    nz = _f64(nz, "nonzeros")
    cols = nz.shape[-1]
    rows = nz.numel() // cols if cols else 0
    pr = None
    if present is not None:
        pr = present.to(device=nz.device, dtype=torch.uint8).expand(nz.shape).contiguous()
    out = torch.empty_like(nz)
    with torch.cuda.device(nz.device):
        _lib.check(_lib.load().dfss_kmod_softmax_nonzeros(_lib.ptr(nz), _lib.ptr(pr), _lib.ptr(out), rows, cols,
                                                          _lib.stream_of(nz)), "softmax_nonzeros")
    return out


def spmm_gather(nz: torch.Tensor, cols: torch.Tensor, present: torch.Tensor | None, v: torch.Tensor) -> torch.Tensor:
    """out[i, :] += nz[i, c] * v[cols[i, c], :] over present c, ascending (_kernels_numba.py:91-106);
    nz / cols / present [rows, nz_cols], v [v_rows, d]."""
    nz, v = _f64(nz, "nonzeros"), _f64(v, "v")
    rows, nzc = nz.shape
    v_rows, d = v.shape
    c = cols.to(device=nz.device, dtype=torch.int64).contiguous()
    pr = None if present is None else present.to(device=nz.device, dtype=torch.uint8).expand(nz.shape).contiguous()
    out = torch.empty((rows, d), dtype=torch.float64, device=nz.device)
    err = torch.full((1,), _INT32_MAX, dtype=torch.int32, device=nz.device)
    with torch.cuda.device(nz.device):
        _lib.check(_lib.load().dfss_kmod_spmm_gather(_lib.ptr(nz), _lib.ptr(c), _lib.ptr(pr), _lib.ptr(v), _lib.ptr(out),
                                                     rows, nzc, v_rows, d, _lib.ptr(err), _lib.stream_of(nz)),
                   "spmm_gather")
    bad = int(err.item())
    if bad != _INT32_MAX:
        raise IndexError(f"spmm_gather: column index out of range [0, {v_rows}) in row {bad}")
    return out


def gemm_abt(a: torch.Tensor, b: torch.Tensor, scale: float) -> torch.Tensor:
    """scale * a @ b.T, one ascending accumulator per element (_kernels_numba.py:16-39)."""
    a, b = _f64(a, "a"), _f64(b, "b")
    n, kdim = a.shape
    m = b.shape[0]
    out = torch.empty((n, m), dtype=torch.float64, device=a.device)
    with torch.cuda.device(a.device):
        _lib.check(_lib.load().dfss_kmod_gemm_abt(_lib.ptr(a), _lib.ptr(b), float(scale), n, m, kdim, _lib.ptr(out),
                                                  _lib.stream_of(a)), "gemm_abt")
    return out


def row_softmax_dense(x: torch.Tensor) -> torch.Tensor:
    """Row-wise stable softmax of [..., cols] (_kernels_numba.py:43-62)."""
    x = _f64(x, "x")
    cols = x.shape[-1]
    rows = x.numel() // cols if cols else 0
    out = torch.empty_like(x)
    with torch.cuda.device(x.device):
        _lib.check(_lib.load().dfss_kmod_row_softmax_dense(_lib.ptr(x), _lib.ptr(out), rows, cols, _lib.stream_of(x)),
                   "row_softmax_dense")
    return out


def batched(fn, *tensors: torch.Tensor, nbatch: int = 2):
    """Apply a 2-D kernel over the leading batch dimensions of `tensors` (each [..., r, c])."""
    batch = tuple(tensors[0].shape[:-nbatch])
    if not batch:
        return fn(*tensors)
    flat = [t.reshape((-1,) + tuple(t.shape[-nbatch:])) for t in tensors]
    outs = [fn(*(f[i] for f in flat)) for i in range(flat[0].shape[0])]
    if isinstance(outs[0], tuple):
        return tuple(torch.stack([o[j] for o in outs]).reshape(batch + tuple(outs[0][j].shape))
                     for j in range(len(outs[0])))
    return torch.stack(outs).reshape(batch + tuple(outs[0].shape))
