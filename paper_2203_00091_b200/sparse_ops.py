"""Operations on compressed matrices: per-row softmax and SpMM (reference: sparse_ops.py)."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .codec import BlockMask, CompressedSparse, Layout
from .dense import DenseMatrix, as_tensor

_INT32_MAX = 2**31 - 1


def softmax_rows(c: CompressedSparse, out_dtype: torch.dtype | None = None, *, check: bool = True) -> CompressedSparse:
    """Stable softmax over each row's kept entries (sparse_ops.py:18-37).

    Rows whose tiles are all masked are rejected ("empty row N"), as is NaN
    input ("NaN") -- the NaN check reads a device flag, i.e. synchronises;
    pass ``check=False`` on hot paths.
    """
    if c.layout is not Layout.LOGICAL:
        raise ValueError("softmax requires the logical layout")
    if c.block_mask is not None:
        bm = c.block_mask
        rows_present = bm.nonzero_keep(c.rows, c.dense_cols).any(axis=1)
        if not rows_present.all():
            row = int(np.flatnonzero(~rows_present)[0])
            raise ValueError(f"empty row {row}: all tiles masked, softmax undefined")
    out_dtype = out_dtype or c.nonzeros.dtype
    if c.nonzeros.dtype == torch.float64:
        # reference arithmetic (_kernels_numba.softmax_nonzeros) on the reference's dtype
        from . import kernels_f64

        present = c.present_nonzeros()
        if check and bool(torch.isnan(c.nonzeros[..., present]).any()):
            raise ValueError("NaN in nonzeros, softmax rejected")
        out = kernels_f64.softmax_nonzeros(c.nonzeros, present).to(out_dtype)
        return CompressedSparse(c.rows, c.dense_cols, c.mode, out, c.meta_hw, layout=Layout.LOGICAL,
                                block_mask=c.block_mask)
    out = torch.empty(c.nonzeros.shape, dtype=out_dtype, device=c.device)
    err = torch.full((2,), _INT32_MAX, dtype=torch.int32, device=c.device) if check else None
    keep = c.block_mask.device_keep(c.device) if c.block_mask is not None else None
    tr = c.block_mask.tile_rows if c.block_mask is not None else 0
    tc = c.block_mask.tile_cols if c.block_mask is not None else 0
    lib = _lib.load()
    with torch.cuda.device(c.device):
        _lib.check(lib.dfss_softmax_rows(_lib.ptr(c.nonzeros), _lib.ptr(out), _lib.dtype_id(c.nonzeros.dtype),
                                         _lib.dtype_id(out_dtype), c.bh, c.rows, c.nonzero_cols, _lib.ptr(keep), tr, tc,
                                         _lib.ptr(err), _lib.stream_of(out)), "softmax_rows")
    if check:
        e = err.tolist()
        if e[1] != _INT32_MAX:
            raise ValueError("NaN in nonzeros, softmax rejected")
        if e[0] != _INT32_MAX:
            raise ValueError(f"empty row {(e[0] - 1) % c.rows}: all tiles masked, softmax undefined")
    return CompressedSparse(c.rows, c.dense_cols, c.mode, out, c.meta_hw, layout=Layout.LOGICAL,
                            block_mask=c.block_mask)


def spmm(a: CompressedSparse, v, block_mask: BlockMask | None = None, out_dtype: torch.dtype | None = None) -> DenseMatrix:
    """decompress(a) @ v with the metadata consumed in place (sparse_ops.py:40-68)."""
    if a.layout is not Layout.LOGICAL:
        raise ValueError("spmm requires the logical layout")
    vt = as_tensor(v)
    if a.dense_cols != vt.shape[-2]:
        raise ValueError(
            f"shape mismatch: sparse operand is {a.rows}x{a.dense_cols}, dense operand has {vt.shape[-2]} rows"
        )
    if block_mask is not None and a.block_mask is not None:
        raise ValueError("block mask given both on the matrix and as an argument")
    bm = block_mask if block_mask is not None else a.block_mask
    if bm is not None:
        bm.check_covers(a.rows, a.dense_cols)
    _lib.require_cuda(vt)
    if tuple(vt.shape[:-2]) != a.batch_shape:
        if vt.dim() == 2 and a.bh == 1:
            pass
        else:
            raise ValueError(f"shape mismatch: batch dims {a.batch_shape} vs {tuple(vt.shape[:-2])}")
    vt = vt.contiguous()
    d = vt.shape[-1]
    out_dtype = out_dtype or torch.promote_types(a.nonzeros.dtype, vt.dtype)
    if a.nonzeros.dtype == torch.float64 or vt.dtype == torch.float64:
        # reference arithmetic (_kernels_numba.spmm_gather): decoded columns, presence mask
        from . import kernels_f64
        from .codec import nonzero_columns

        a_m = a if a.block_mask is not None or bm is None else CompressedSparse(
            a.rows, a.dense_cols, a.mode, a.nonzeros, a.meta_hw, layout=a.layout, block_mask=bm)
        cols = nonzero_columns(a_m)
        present = cols >= 0
        v64 = vt.to(torch.float64).expand(a.batch_shape + tuple(vt.shape[-2:])) if vt.dim() == 2 else vt.to(torch.float64)
        out = kernels_f64.batched(lambda p, c_, pr, v_: kernels_f64.spmm_gather(p, c_, pr, v_),
                                  a.nonzeros.to(torch.float64), cols, present.expand(cols.shape), v64)
        return DenseMatrix(out.to(out_dtype), check_finite=False)
    out = torch.empty(a.batch_shape + (a.rows, d), dtype=out_dtype, device=a.device)
    keep = bm.device_keep(a.device) if bm is not None else None
    tr = bm.tile_rows if bm is not None else 0
    tc = bm.tile_cols if bm is not None else 0
    lib = _lib.load()
    with torch.cuda.device(a.device):
        _lib.check(lib.dfss_spmm(_lib.ptr(a.nonzeros), _lib.ptr(a.meta_hw), _lib.ptr(vt), _lib.ptr(out), a.mode.group_size,
                                 _lib.dtype_id(a.nonzeros.dtype), _lib.dtype_id(vt.dtype), _lib.dtype_id(out_dtype), a.bh,
                                 a.rows, a.dense_cols, d, _lib.ptr(keep), tr, tc, None, _lib.stream_of(out)), "spmm")
    return DenseMatrix(out, check_finite=False)


def spmm_softmax(a: CompressedSparse, v, out_dtype: torch.dtype | None = None) -> DenseMatrix:
    """``spmm(softmax_rows(a), v)`` in one kernel: the row softmax is applied to each staged
    P tile in shared memory (exp(s - row max)) and the output rows are divided by the row
    sums -- no HBM round trip for the probabilities.  Needs ``a`` from
    ``sddmm_prune(..., with_row_max=True)`` (tcgen05 path: 2:4 or 1:2, 16-bit, d = 64)."""
    if a.row_max is None:
        raise ValueError("spmm_softmax needs the row maxima: call sddmm_prune(..., with_row_max=True)")
    if a.layout is not Layout.LOGICAL or a.block_mask is not None:
        raise ValueError("spmm_softmax requires the logical layout without a block mask")
    vt = as_tensor(v)
    if a.dense_cols != vt.shape[-2]:
        raise ValueError(
            f"shape mismatch: sparse operand is {a.rows}x{a.dense_cols}, dense operand has {vt.shape[-2]} rows"
        )
    _lib.require_cuda(vt)
    vt = vt.contiguous()
    d = vt.shape[-1]
    out_dtype = out_dtype or vt.dtype
    out = torch.empty(a.batch_shape + (a.rows, d), dtype=out_dtype, device=a.device)
    lib = _lib.load()
    with torch.cuda.device(a.device):
        _lib.check(lib.dfss_spmm(_lib.ptr(a.nonzeros), _lib.ptr(a.meta_hw), _lib.ptr(vt), _lib.ptr(out), a.mode.group_size,
                                 _lib.dtype_id(a.nonzeros.dtype), _lib.dtype_id(vt.dtype), _lib.dtype_id(out_dtype), a.bh,
                                 a.rows, a.dense_cols, d, None, 0, 0, _lib.ptr(a.row_max), _lib.stream_of(out)),
                   "spmm_softmax")
    return DenseMatrix(out, check_finite=False)
