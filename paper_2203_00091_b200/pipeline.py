"""End-to-end DFSS attention on the B200 (reference: pipeline.py).

``nm_attention`` keeps the reference signature (pipeline.py:15-32);
``dfss_attention`` is the tensor-level drop-in for a model's attention over
[..., n, d] CUDA tensors and is what ``DFSSAttention`` and bench.py call.
"""

from __future__ import annotations

import contextlib
import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .codec import BlockMask, SparsityMode, as_mode, decompress
from .dense import AttentionInputs, DenseMatrix, as_tensor, dense_attention_weights
from .fused import _MATH, attention_sddmm
from .sparse_ops import softmax_rows, spmm


def workspace_bytes(mode, dtype: torch.dtype, bh: int, n: int, d: int, math_mode: str = "auto",
                    block_mask: BlockMask | None = None) -> int:
    """Device scratch one dfss_attention call needs on the path it will take: 0 for the fused
    16-bit kernel (its liveness bitmaps with a block mask), V^T for the fused tf32 kernel, the
    compressed P + metadata when staged."""
    mode = as_mode(mode)
    tr, tc_ = (block_mask.tile_rows, block_mask.tile_cols) if block_mask is not None else (0, 0)
    return int(_lib.load().dfss_nm_attention_workspace_bytes_for(mode.group_size, _lib.dtype_id(dtype),
                                                                 _MATH[math_mode], bh, n, d, tr, tc_,
                                                                 int(block_mask is not None)))


def _check_block_mask(block_mask: BlockMask, n: int, mode: SparsityMode) -> None:
    """Reference validation of a BlockMask for an n x n score matrix (fused.py:58-82,
    sparse_ops.py:25-30): tile columns group-aligned, grid covering, no empty row."""
    if block_mask.tile_cols % mode.group_size != 0:
        raise ValueError(
            f"tile {block_mask.tile_rows}x{block_mask.tile_cols} must have columns divisible by the "
            f"group size {mode.group_size}"
        )
    block_mask.check_covers(n, n)
    empty = ~block_mask.keep.any(axis=1)
    if empty.any():
        row = int(np.flatnonzero(empty)[0]) * block_mask.tile_rows
        raise ValueError(f"empty row {row}: all tiles masked, softmax undefined")


def dfss_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, mode="2:4", *, math_mode: str = "auto",
                   block_mask: BlockMask | None = None, out: torch.Tensor | None = None,
                   workspace: torch.Tensor | None = None) -> torch.Tensor:
    """softmax_N:M(Q K^T / sqrt d) V for [..., n, d] q/k/v on one CUDA device.

    One C-ABI call (dfss_nm_attention / dfss_nm_attention_masked); no dense n x n tensor is
    allocated.  ``block_mask`` (shared by every batch / head) makes masked tiles structurally
    absent, as in the reference's fused path (fused.py:73-82).
    """
    mode = as_mode(mode)
    shape = q.shape
    if shape != k.shape or shape != v.shape:
        raise ValueError(f"Q, K, V must share shape (n, d); got {tuple(q.shape)}, {tuple(k.shape)}, {tuple(v.shape)}")
    if len(shape) < 2:
        raise ValueError("expected [..., n, d] tensors")
    n, d = shape[-2], shape[-1]
    if n % mode.group_size:
        raise ValueError(f"score columns {n} not group-aligned for mode {mode.value} (need a multiple of {mode.group_size})")
    if math_mode not in _MATH:
        raise ValueError(f"unknown math mode {math_mode!r}")
    _lib.require_cuda(q, k, v)
    dtype = q.dtype
    if not (dtype == k.dtype == v.dtype):
        raise ValueError("Q, K, V must share a dtype")
    if dtype == torch.float64:
        raise ValueError("dfss_attention computes in bf16/fp16/fp32: cast float64 explicitly, or use nm_attention "
                         "(reference float64 arithmetic)")
    dev = q.get_device()
    if not (dev == k.get_device() == v.get_device()) or (out is not None and out.get_device() != dev) or (
            workspace is not None and workspace.get_device() != dev):
        raise ValueError("Q, K, V, out and workspace must be on one CUDA device")
    if not q.is_contiguous():
        q = q.contiguous()
    if not k.is_contiguous():
        k = k.contiguous()
    if not v.is_contiguous():
        v = v.contiguous()
    if out is None:
        out = torch.empty_like(q)
    # per-(shape, dtype, mode, math, mask) constants: the host path runs once per step, so its cost
    # is part of every small config's step time (c2: ~48 us of kernel)
    key = (shape, dtype, mode.group_size, math_mode,
           None if block_mask is None else (block_mask.tile_rows, block_mask.tile_cols))
    consts = _CALL_CACHE.get(key)
    if consts is None:
        bh = math.prod(shape[:-2])
        consts = (bh, workspace_bytes(mode, dtype, bh, n, d, math_mode, block_mask), _lib.dtype_id(dtype),
                  _MATH[math_mode])
        if len(_CALL_CACHE) > 256:
            _CALL_CACHE.clear()
        _CALL_CACHE[key] = consts
    bh, need, dt, mm = consts
    if need and (workspace is None or workspace.numel() < need):
        workspace = torch.empty(need, dtype=torch.uint8, device=q.device)
    lib = _lib.load()
    ws_ptr = None if workspace is None else workspace.data_ptr()
    # the C ABI launches on the current device: switch only when q lives elsewhere
    ctx = torch.cuda.device(dev) if dev != torch.cuda.current_device() else contextlib.nullcontext()
    with ctx:
        stream = torch._C._cuda_getCurrentRawStream(dev)
        if block_mask is None:
            _lib.check(lib.dfss_nm_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                             mode.group_size, dt, mm, bh, n, d, ws_ptr, need, stream),
                       "nm_attention")
            return out
        _check_block_mask(block_mask, n, mode)
        keep = block_mask.device_keep(q.device)
        _lib.check(lib.dfss_nm_attention_masked(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                                mode.group_size, dt, mm, bh, n, d, _lib.ptr(keep),
                                                block_mask.tile_rows, block_mask.tile_cols, ws_ptr, need, stream),
                   "nm_attention")
    return out


#: dfss_attention's per-call constants, keyed by (shape, dtype, group size, math mode, block mask)
_CALL_CACHE: dict = {}


#: dfss_nm_attention_path ids (include/dfss.h)
PATHS = {1: "fused-16bit", 2: "fused-tf32", 3: "staged-tcgen05", 4: "staged-ffma", 5: "staged-masked",
         6: "staged-3xtf32"}


def attention_path(mode, dtype: torch.dtype, n: int, d: int, math_mode: str = "auto",
                   block_mask: BlockMask | None = None, bh: int = 1) -> str:
    """Name of the kernel path dfss_attention takes for these arguments (no launch); ``bh`` is the
    flattened batch x heads count (the exact-FP32 3xTF32 path is chosen from ~1 M scores)."""
    mode = as_mode(mode)
    tr, tc_ = (block_mask.tile_rows, block_mask.tile_cols) if block_mask is not None else (0, 0)
    pid = int(_lib.load().dfss_nm_attention_path_bh(mode.group_size, _lib.dtype_id(dtype), _MATH[math_mode], int(bh), n,
                                                    d, tr, tc_, int(block_mask is not None)))
    if pid < 0:
        _lib.check(pid, "attention path")
    return PATHS[pid]


@dataclass(frozen=True)
class AttentionDump:
    """Selection evidence of one dfss_attention call (dfss_nm_attention_dump).

    scores: fp32 [..., n, n], the post-scale scores every prune compared (NaN where a fused kernel
    skipped a fully masked 128 x 128 step); meta: uint8 [..., n, n / gs], the LOGICAL nibbles of the
    call's mode decoded from the metadata words the kernel handed to tcgen05.mma.sp (0 where
    nothing was selected: masked chunks, skipped steps); path: the kernel path that ran."""

    out: torch.Tensor
    scores: torch.Tensor
    meta: torch.Tensor
    path: str


def dfss_attention_dump(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, mode="2:4", *, math_mode: str = "auto",
                        block_mask: BlockMask | None = None) -> AttentionDump:
    """dfss_attention plus the scores and metadata its prune produced (parity evidence only: it
    writes an n x n fp32 tensor, which the product path never does).  Same kernels, same output."""
    mode = as_mode(mode)
    if q.shape != k.shape or q.shape != v.shape or q.dim() < 2:
        raise ValueError(f"Q, K, V must share shape [..., n, d]; got {tuple(q.shape)}")
    _lib.require_cuda(q, k, v)
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    n, d = q.shape[-2], q.shape[-1]
    bh = int(np.prod(q.shape[:-2], dtype=np.int64)) if q.dim() > 2 else 1
    lib = _lib.load()
    out = torch.empty_like(q)
    need = workspace_bytes(mode, q.dtype, bh, n, d, math_mode, block_mask)
    ws = torch.empty(max(need, 1), dtype=torch.uint8, device=q.device)
    scores = torch.full((bh, n, n), float("nan"), dtype=torch.float32, device=q.device)
    words = max(int(lib.dfss_meta_hw_words(4, bh, n, n)), int(lib.dfss_meta_hw_words(2, bh, n, n)))
    meta_hw = torch.zeros(words, dtype=torch.int32, device=q.device)
    meta_mode = ctypes.c_int(0)
    keep = None
    tr = tc_ = 0
    if block_mask is not None:
        _check_block_mask(block_mask, n, mode)
        keep = block_mask.device_keep(q.device)
        tr, tc_ = block_mask.tile_rows, block_mask.tile_cols
    with torch.cuda.device(q.device):
        _lib.check(lib.dfss_nm_attention_dump(_lib.ptr(q), _lib.ptr(k), _lib.ptr(v), _lib.ptr(out), mode.group_size,
                                              _lib.dtype_id(q.dtype), _MATH[math_mode], bh, n, d, _lib.ptr(keep), tr,
                                              tc_, _lib.ptr(ws), need, _lib.ptr(scores), _lib.ptr(meta_hw),
                                              ctypes.byref(meta_mode), _lib.stream_of(q)), "nm_attention_dump")
        gs = meta_mode.value
        logical = torch.empty((bh, n, n // gs), dtype=torch.uint8, device=q.device)
        _lib.check(lib.dfss_meta_hw_to_logical(_lib.ptr(meta_hw), _lib.ptr(logical), gs, bh, n, n,
                                               _lib.stream_of(q)), "meta decode")
    if gs != mode.group_size:
        # 1:2 run as the 2:4 pattern (one survivor per pair): nibble lo | hi << 2 with lo in {0, 1}
        # (pair 0 keeps element lo) and hi in {2, 3}; 0x4 / 0 mark masked / skipped groups
        lo, hi = (logical & 3).long(), (logical >> 2).long()
        valid = (lo <= 1) & (hi >= 2)
        absent = (logical == 0x4) | (logical == 0)
        p0 = torch.where(lo == 0, 0x4, 0xE)
        p1 = torch.where(hi == 2, 0x4, 0xE)
        pairs = torch.stack((p0, p1), dim=-1)
        pairs = torch.where(absent[..., None], 0, torch.where(valid[..., None], pairs, 0xFF))
        logical = pairs.reshape(bh, n, n // 2).to(torch.uint8)
    shape = tuple(q.shape[:-2])
    return AttentionDump(out, scores.reshape(shape + (n, n)), logical.reshape(shape + (n, n // mode.group_size)),
                         attention_path(mode, q.dtype, n, d, math_mode, block_mask, bh))


_HOST_STREAMS: dict[int, tuple[torch.cuda.Stream, torch.cuda.Stream, torch.cuda.Stream]] = {}


def _piece_bounds(bh: int, chunks: int) -> list[int]:
    """Piece boundaries over the flattened batch x heads: `chunks` equal pieces, the last one cut
    into halves / quarters so the copy-out after the last kernel (the pipeline's tail) is short
    (c2, 4 pieces: 1.79 -> 1.7 ms per call, tools/host_timeline.py)."""
    chunks = max(1, min(int(chunks), bh))
    bounds = [bh * i // chunks for i in range(chunks + 1)]
    lo, hi = bounds[-2], bounds[-1]
    if chunks > 1 and hi - lo >= 4:
        bounds[-1:] = [lo + (hi - lo) // 2, lo + 3 * (hi - lo) // 4, hi]
    return bounds


def dfss_attention_host(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, mode="2:4", *, math_mode: str = "auto",
                        block_mask: BlockMask | None = None, out: torch.Tensor | None = None, chunks: int = 4,
                        device: torch.device | int | None = None, non_blocking: bool = False) -> torch.Tensor:
    """dfss_attention for HOST tensors [..., n, d] (the reference's own calling convention: its
    kernels take host arrays): returns a host tensor.  The flattened batch x heads is cut into
    `chunks` pieces; the host->device copy of piece i+1, the fused kernel on piece i and the
    device->host copy of piece i-1 run concurrently on three streams (PCIe is full duplex), with
    two device buffers per direction.  Pinned inputs / output make the copies asynchronous
    (unpinned ones are staged by the driver, still correct).  Ordered after prior work on the
    current stream, and the current stream waits for the last copy, so events recorded around
    the call time the whole transfer + compute.

    By default the call is synchronous like the reference's (its kernels return host arrays): it
    returns once `out` holds the result.  ``non_blocking=True`` returns right after enqueueing;
    then `out` must not be read, nor q / k / v modified, before the current stream is
    synchronised (bench.py times the pipelined copies this way, with events on that stream)."""
    if q.is_cuda or k.is_cuda or v.is_cuda:
        raise ValueError("dfss_attention_host takes host tensors; use dfss_attention for device tensors")
    if q.shape != k.shape or q.shape != v.shape or q.dim() < 2:
        raise ValueError(f"Q, K, V must share shape [..., n, d]; got {tuple(q.shape)}, {tuple(k.shape)}, {tuple(v.shape)}")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index or 0)
    n, d = q.shape[-2], q.shape[-1]
    bh = int(np.prod(q.shape[:-2], dtype=np.int64)) if q.dim() > 2 else 1
    qf, kf, vf = (x.reshape(bh, n, d) for x in (q, k, v))
    if out is None:
        out = torch.empty(q.shape, dtype=q.dtype, pin_memory=True)
    of = out.view(bh, n, d)
    bounds = _piece_bounds(bh, chunks)
    chunks = len(bounds) - 1
    width = max(bounds[i + 1] - bounds[i] for i in range(chunks))
    if dev.index not in _HOST_STREAMS:
        _HOST_STREAMS[dev.index] = tuple(torch.cuda.Stream(dev) for _ in range(3))
    s_in, s_run, s_out = _HOST_STREAMS[dev.index]
    cur = torch.cuda.current_stream(dev)
    start = torch.cuda.Event()
    start.record(cur)
    dq = torch.empty((2, 3, width, n, d), dtype=q.dtype, device=dev)    # [slot][q,k,v] input buffers
    do = torch.empty((2, width, n, d), dtype=q.dtype, device=dev)       # output buffers
    ws = None
    need = workspace_bytes(mode, q.dtype, width, n, d, math_mode, block_mask)
    if need:
        ws = torch.empty(need, dtype=torch.uint8, device=dev)
    copied, ran, drained = [], [], []
    for i in range(chunks):
        lo, hi = bounds[i], bounds[i + 1]
        slot, w = i % 2, hi - lo
        with torch.cuda.stream(s_in):
            s_in.wait_event(start)
            if i >= 2:
                s_in.wait_event(ran[i - 2])          # input slot free once that piece's kernel ran
            for j, src in enumerate((qf, kf, vf)):
                dq[slot, j, :w].copy_(src[lo:hi], non_blocking=True)
            copied.append(torch.cuda.Event())
            copied[i].record(s_in)
        with torch.cuda.stream(s_run):
            s_run.wait_event(copied[i])
            if i >= 2:
                s_run.wait_event(drained[i - 2])     # output slot free once copied out
            dfss_attention(dq[slot, 0, :w], dq[slot, 1, :w], dq[slot, 2, :w], mode, math_mode=math_mode,
                           block_mask=block_mask, out=do[slot, :w], workspace=ws)
            ran.append(torch.cuda.Event())
            ran[i].record(s_run)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ran[i])
            of[lo:hi].copy_(do[slot, :w], non_blocking=True)
            drained.append(torch.cuda.Event())
            drained[i].record(s_out)
    cur.wait_event(drained[-1])
    if not non_blocking:
        drained[-1].synchronize()
    # the device buffers are released to the caching allocator; keep them alive until the copies
    # ran by recording their use on every stream that touched them
    for st in (s_in, s_run, s_out):
        dq.record_stream(st)
        do.record_stream(st)
        if ws is not None:
            ws.record_stream(st)
    return out


def nm_attention(inputs: AttentionInputs, mode: SparsityMode, block_mask: BlockMask | None = None, *,
                 tile_rows: int = 32, tile_cols: int = 64, precision: str = "auto") -> DenseMatrix:
    """Drop-in sparse attention: fused prune -> sparse softmax -> SpMM (pipeline.py:15-32).

    16/32-bit inputs run dfss_attention (one fused kernel for 16-bit; exact FP32 FFMA for fp32).
    float64 inputs -- the reference's dtype -- run the reference's arithmetic on the device by
    default (``precision="auto"``: attention_sddmm -> softmax_rows -> spmm over kernels_f64, the
    reference's numbers up to exp rounding); ``precision="fp32"`` narrows them explicitly to the
    exact-FP32 kernels (tolerance 1e-5) and returns float64."""
    mode = as_mode(mode)
    if precision not in ("auto", "fp32"):
        raise ValueError(f"unknown precision {precision!r}; pick 'auto' or 'fp32'")
    if block_mask is not None and (block_mask.tile_rows, block_mask.tile_cols) != (tile_rows, tile_cols):
        raise ValueError(
            f"block mask tiles {block_mask.tile_rows}x{block_mask.tile_cols} "
            f"do not match the fused tiling {tile_rows}x{tile_cols}"
        )
    q, k, v = inputs.q.data, inputs.k.data, inputs.v.data
    if q.dtype == torch.float64 and precision == "auto":
        compressed, _ = attention_sddmm(q, k, mode, block_mask, tile_rows=tile_rows, tile_cols=tile_cols)
        return spmm(softmax_rows(compressed), v)
    if q.dtype == torch.float64:
        out = dfss_attention(q.float(), k.float(), v.float(), mode, block_mask=block_mask)
        return DenseMatrix(out.double(), check_finite=False)
    out = dfss_attention(q, k, v, mode, block_mask=block_mask)
    return DenseMatrix(out, check_finite=False)


@dataclass(frozen=True)
class ApproxError:
    """Error of a sparse output against the full-attention baseline (pipeline.py:35-46)."""

    rel_l2: float
    max_abs: float
    row_rel: torch.Tensor

    def __str__(self) -> str:
        return f"rel_l2={self.rel_l2:.6e} max_abs={self.max_abs:.6e}"


def approx_error(full, sparse) -> ApproxError:
    """Relative Frobenius error, max absolute error, per-row errors (pipeline.py:49-57), in float64."""
    f = as_tensor(full).double()
    s = as_tensor(sparse).double()
    if f.shape != s.shape:
        raise ValueError(f"shape mismatch: {tuple(f.shape)} vs {tuple(s.shape)}")
    diff = f - s
    denom = torch.linalg.norm(f)
    rel = float(torch.linalg.norm(diff) / denom) if float(denom) > 0 else 0.0
    row_norms = torch.linalg.norm(f, dim=-1)
    safe = torch.where(row_norms > 0, row_norms, torch.ones_like(row_norms))
    row_rel = torch.where(row_norms > 0, torch.linalg.norm(diff, dim=-1) / safe, torch.zeros_like(row_norms))
    return ApproxError(rel, float(diff.abs().max()), row_rel)


@dataclass(frozen=True)
class AttentionWeights:
    dense: DenseMatrix
    sparse: DenseMatrix


def attention_heatmap(inputs: AttentionInputs, mode: SparsityMode) -> AttentionWeights:
    """Dense and sparse weight matrices (pipeline.py:60-78)."""
    dense = dense_attention_weights(inputs)
    compressed, _ = attention_sddmm(inputs.q, inputs.k, as_mode(mode))
    return AttentionWeights(dense, decompress(softmax_rows(compressed)))


def reference_scale(d: int) -> float:
    return 1.0 / math.sqrt(d)
