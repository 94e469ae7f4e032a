"""CUDA kernel module for the reference package ``nmattn`` 0.1.0 (drop-in backend).

The reference dispatches its hot loops through a duck-typed kernel module returned by
``backend.kernels()`` (``pkg/src/nmattn/backend.py:63-67``), implemented twice in the reference
(``_kernels_numba.py:39,62,87,106,188`` and ``_kernels_numpy.py:18-79``).  This file is a third
implementation of the same five functions with the same signatures, argument meaning and return
values, computed on the B200 by libdfss_sm100a.so (include/dfss.h, ``dfss_kmod_*``):

* ``sddmm_compress(q, kmat, scale, group_size, tile_rows, tile_cols, keep)
  -> (nonzeros, meta, peak, nnz, nib)``
* ``softmax_nonzeros(nz, present) -> out``
* ``spmm_gather(nz, cols, present, v) -> out``
* ``gemm_abt(a, b, scale, tile_rows, tile_cols, k_panel) -> out``
* ``row_softmax_dense(x) -> out``

Conventions kept from the reference kernels: float64 C-contiguous numpy arrays in, freshly
allocated numpy arrays out, inputs never mutated, no validation beyond what the reference's own
wrappers already did (fused.py:58-82, sparse_ops.py:25-32, dense.py:96-101), synchronous.  The
arithmetic is the reference's: float64, one accumulator per output, ascending reduction index,
products and sums separately rounded (numba runs with fastmath off), so sddmm_compress,
spmm_gather and gemm_abt return bitwise the numba results and the softmaxes differ only through
exp (<= 1 ulp).

To plug it in, copy this file to ``nmattn/_kernels_cuda.py`` and add ``"cuda"`` to
``backend._VALID`` (INTEGRATION.md §1 shows the one-line diff); ``paper_2203_00091_b200`` must be
importable and a B200 present.  There is no CPU fallback: without the library or a device every
call raises.
"""

from __future__ import annotations

import numpy as np
import torch

from paper_2203_00091_b200 import kernels_f64 as _k


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("nmattn cuda backend: no CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(a: np.ndarray, dtype) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).to(_dev())


def _host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy()


def sddmm_compress(q, kmat, scale, group_size, tile_rows, tile_cols, keep):
    """Fused score -> prune -> compress (_kernels_numba.py:110-188)."""
    n = q.shape[0]
    m = kmat.shape[0]
    keep = np.asarray(keep, dtype=bool)
    nz, meta = _k.sddmm_compress(_to_dev(q, np.float64), _to_dev(kmat, np.float64), scale, group_size, tile_rows,
                                 tile_cols, keep)
    # structural counters (_kernels_numba.py:126-184): over the kept tiles, peak tile area,
    # nonzeros written (2 per 2:4 group, 1 per 1:2 group) and nibbles written
    peak = nnz = nib = 0
    for ti, tj in np.argwhere(keep):
        ih = min((ti + 1) * tile_rows, n) - ti * tile_rows
        jw = min((tj + 1) * tile_cols, m) - tj * tile_cols
        peak = max(peak, ih * jw)
        groups = max(ih, 0) * max(jw // group_size, 0)
        nib += groups
        nnz += groups * (2 if group_size == 4 else 1)
    return _host(nz), _host(meta), peak, nnz, nib


def softmax_nonzeros(nz, present):
    """Per-row stable softmax over present nonzeros (_kernels_numba.py:66-87)."""
    return _host(_k.softmax_nonzeros(_to_dev(nz, np.float64), _to_dev(np.asarray(present, dtype=bool), np.bool_)))


def spmm_gather(nz, cols, present, v):
    """out[i, :] += nz[i, c] * v[cols[i, c], :] over present c, ascending (_kernels_numba.py:91-106)."""
    return _host(_k.spmm_gather(_to_dev(nz, np.float64), _to_dev(cols, np.int64),
                                _to_dev(np.asarray(present, dtype=bool), np.bool_), _to_dev(v, np.float64)))


def gemm_abt(a, b, scale, tile_rows, tile_cols, k_panel):
    """out = scale * a @ b.T with one ascending accumulator per element (_kernels_numba.py:16-39);
    the tiling arguments only reorder the reference's traversal and do not change the result."""
    return _host(_k.gemm_abt(_to_dev(a, np.float64), _to_dev(b, np.float64), scale))


def row_softmax_dense(x):
    """Row-wise stable softmax of a dense matrix (_kernels_numba.py:43-62)."""
    return _host(_k.row_softmax_dense(_to_dev(x, np.float64)))


__all__ = ["sddmm_compress", "softmax_nonzeros", "spmm_gather", "gemm_abt", "row_softmax_dense"]
