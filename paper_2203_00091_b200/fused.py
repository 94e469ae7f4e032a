"""Score computation fused with pruning and compression (reference: fused.py).

``sddmm_prune`` produces the compressed scores straight from Q and K: the
tcgen05 (16-bit) or FP32-FFMA (fp32) kernel keeps each score tile in TMEM /
registers, prunes it in its epilogue, and writes only nonzeros and metadata.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .codec import BlockMask, CompressedSparse, SparsityMode, _meta_words_host, as_mode
from .dense import as_tensor

_MATH = {"auto": _lib.MATH_AUTO, "ffma": _lib.MATH_FFMA, "tf32": _lib.MATH_TF32}


@dataclass(frozen=True)
class FusedStats:
    """Structural accounting for one fused run, per (batch, head) (fused.py:22-38)."""

    peak_tile_elems: int
    dense_elems_written: int
    nonzeros_written: int
    nibbles_written: int

    def __post_init__(self) -> None:
        if self.dense_elems_written != 0:
            raise ValueError("fused path must not write dense score elements")


def _stats(n: int, m: int, gs: int, tile_rows: int, tile_cols: int, keep: np.ndarray | None) -> FusedStats:
    """The reference kernel's counters (_kernels_numba.py:117-184) from the tile grid."""
    gr, gc = -(-n // tile_rows), -(-m // tile_cols)
    ih = np.minimum(np.arange(gr) * tile_rows + tile_rows, n) - np.arange(gr) * tile_rows
    jw = np.minimum(np.arange(gc) * tile_cols + tile_cols, m) - np.arange(gc) * tile_cols
    area = ih[:, None] * jw[None, :]
    k = np.ones((gr, gc), dtype=bool) if keep is None else keep
    peak = int(area[k].max()) if k.any() else 0
    nnz = int((ih[:, None] * (jw[None, :] // gs) * (gs // 2) * k).sum()) if gs == 4 else int(
        (ih[:, None] * (jw[None, :] // 2) * k).sum())
    nib = int((ih[:, None] * (jw[None, :] // gs) * k).sum())
    return FusedStats(peak_tile_elems=peak, dense_elems_written=0, nonzeros_written=nnz, nibbles_written=nib)


def sddmm_prune(
    q,
    k,
    mode: SparsityMode,
    scale: float,
    block_mask: BlockMask | None = None,
    *,
    tile_rows: int = 32,
    tile_cols: int = 64,
    nz_dtype: torch.dtype | None = None,
    math_mode: str = "auto",
    scores_out: torch.Tensor | None = None,
    with_row_max: bool = False,
) -> tuple[CompressedSparse, FusedStats]:
    """compress(Q K^T * scale) without materialising the scores (fused.py:41-96).

    q: [..., n, d], k: [..., m, d] CUDA tensors (or DenseMatrix).  Selection
    is bit-exact to the reference rule on the fp32 post-scale scores the
    epilogue sees; ``scores_out`` (fp32 [..., n, m]) receives exactly those
    scores for parity checks (it is the only dense write, off by default).
    ``with_row_max`` also records each row's maximum (tcgen05 path), which lets
    ``spmm_softmax`` fuse the row softmax into the SpMM.
    """
    mode = as_mode(mode)
    qt, kt = as_tensor(q), as_tensor(k)
    if qt.shape[-1] != kt.shape[-1]:
        raise ValueError(f"shape mismatch: Q has d={qt.shape[-1]}, K has d={kt.shape[-1]}")
    if qt.shape[:-2] != kt.shape[:-2]:
        raise ValueError(f"shape mismatch: batch dims {tuple(qt.shape[:-2])} vs {tuple(kt.shape[:-2])}")
    n, m, d = qt.shape[-2], kt.shape[-2], qt.shape[-1]
    gs = mode.group_size
    if m % gs != 0:
        raise ValueError(
            f"score columns {m} not group-aligned for mode {mode.value} (need a multiple of {gs})"
        )
    if tile_cols % gs != 0 or tile_rows < 1:
        raise ValueError(
            f"tile {tile_rows}x{tile_cols} must have columns divisible by the group size {gs}"
        )
    keep = None
    if block_mask is not None:
        if (block_mask.tile_rows, block_mask.tile_cols) != (tile_rows, tile_cols):
            raise ValueError(
                f"block mask tiles {block_mask.tile_rows}x{block_mask.tile_cols} "
                f"do not match the fused tiling {tile_rows}x{tile_cols}"
            )
        block_mask.check_covers(n, m)
        keep = block_mask.keep
    if math_mode not in _MATH:
        raise ValueError(f"unknown math mode {math_mode!r}; pick one of {tuple(_MATH)}")
    _lib.require_cuda(qt, kt)
    if qt.dtype != kt.dtype:
        raise ValueError(f"Q and K dtypes differ ({qt.dtype} vs {kt.dtype})")
    if qt.dtype == torch.float64:
        # the reference's own dtype: its arithmetic on the device (kernels_f64, bitwise the numba
        # sddmm_compress), not a rounded fp32 approximation
        if math_mode == "tf32" or scores_out is not None or with_row_max:
            raise ValueError("float64 inputs run the reference arithmetic: no tf32, scores_out or row maxima")
        from . import kernels_f64

        nz, meta = kernels_f64.batched(
            lambda a, b: kernels_f64.sddmm_compress(a, b, scale, gs, tile_rows, tile_cols, keep), qt, kt)
        if nz_dtype is not None and nz_dtype != torch.float64:
            nz = nz.to(nz_dtype)
        compressed = CompressedSparse.from_logical(n, m, mode, nz, meta, block_mask=block_mask)
        return compressed, _stats(n, m, gs, tile_rows, tile_cols, keep)
    qt, kt = qt.contiguous(), kt.contiguous()
    batch = tuple(qt.shape[:-2])
    bh = int(np.prod(batch, dtype=np.int64)) if batch else 1
    nz_dtype = nz_dtype or qt.dtype
    nz = torch.empty(batch + (n, m // 2), dtype=nz_dtype, device=qt.device)
    meta = torch.empty(batch + (_meta_words_host(mode, n, m),), dtype=torch.int32, device=qt.device)
    if scores_out is not None:
        if scores_out.dtype != torch.float32 or tuple(scores_out.shape) != batch + (n, m) or not scores_out.is_contiguous():
            raise ValueError("scores_out must be a contiguous float32 tensor of shape (..., n, m)")
    dev_keep = block_mask.device_keep(qt.device) if block_mask is not None else None
    row_max = torch.empty(batch + (n, 4), dtype=torch.float32, device=qt.device) if with_row_max else None
    lib = _lib.load()
    with torch.cuda.device(qt.device):
        _lib.check(
            lib.dfss_sddmm_prune(_lib.ptr(qt), _lib.ptr(kt), _lib.ptr(nz), _lib.ptr(meta), float(scale), gs,
                                 _lib.dtype_id(qt.dtype), _lib.dtype_id(nz_dtype), _MATH[math_mode], bh, n, m, d,
                                 _lib.ptr(dev_keep), tile_rows, tile_cols, _lib.ptr(scores_out), _lib.ptr(row_max),
                                 _lib.stream_of(qt)),
            "sddmm_prune",
        )
    compressed = CompressedSparse(n, m, mode, nz, meta, block_mask=block_mask, row_max=row_max)
    return compressed, _stats(n, m, gs, tile_rows, tile_cols, keep)


def attention_sddmm(q, k, mode: SparsityMode, block_mask: BlockMask | None = None, *, tile_rows: int = 32,
                    tile_cols: int = 64, **kw) -> tuple[CompressedSparse, FusedStats]:
    """Fused scores at the attention scale 1/sqrt(d) (fused.py:99-112)."""
    d = as_tensor(q).shape[-1]
    return sddmm_prune(q, k, mode, 1.0 / math.sqrt(d), block_mask, tile_rows=tile_rows, tile_cols=tile_cols, **kw)
