"""N:M types and the compressed format on the GPU (reference: codec.py).

Same names, argument meaning and ValueError fragments as nmattn.codec
(codec.py:34-372), with device tensors batched over leading dimensions
instead of 2-D float64 arrays.  Compressed nonzeros are stored row-major in
the reference's LOGICAL order; metadata is stored as ``meta_hw`` words, the
tcgen05.mma.sp lane layout documented in include/dfss.h, and decoded to the
reference's logical nibble stream on demand (``CompressedSparse.metadata``).
The Ampere tile-interleaved layout (codec.py:379-441) is not provided: it is
the sm_80 metadata order and has no meaning for tcgen05.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np
import torch

from . import _lib

GROUP_SLOTS = 4


class SparsityMode(enum.Enum):
    """Which N:M pattern is in force (codec.py:34-64)."""

    ONE_OF_TWO = "1:2"
    TWO_OF_FOUR = "2:4"

    @classmethod
    def parse(cls, text: str) -> "SparsityMode":
        for mode in cls:
            if mode.value == text:
                return mode
        raise ValueError(f"unknown sparsity mode {text!r} (expected '1:2' or '2:4')")

    @property
    def group_size(self) -> int:
        return 2 if self is SparsityMode.ONE_OF_TWO else 4

    @property
    def kept_per_group(self) -> int:
        return 1 if self is SparsityMode.ONE_OF_TWO else 2

    @property
    def slots_per_element(self) -> int:
        return 2 if self is SparsityMode.ONE_OF_TWO else 1

    @property
    def admissible_nibbles(self) -> frozenset[int]:
        if self is SparsityMode.ONE_OF_TWO:
            return frozenset({0x4, 0xE})
        return frozenset({0x4, 0x8, 0x9, 0xC, 0xD, 0xE})


def as_mode(mode) -> SparsityMode:
    if isinstance(mode, SparsityMode):
        return mode
    return SparsityMode.parse(str(mode))


class Layout(enum.Enum):
    LOGICAL = "logical"
    TILE_INTERLEAVED = "tile-interleaved"


def nibble_for_slots(lo: int, hi: int) -> int:
    """codec.py:72-76."""
    if not (0 <= lo < hi < GROUP_SLOTS):
        raise ValueError(f"slot pair ({lo}, {hi}) must be strictly increasing in [0, 4)")
    return lo | (hi << 2)


def slots_for_nibble(nibble: int) -> tuple[int, int]:
    """codec.py:79-85."""
    lo = nibble & 0x3
    hi = (nibble >> 2) & 0x3
    if not (0 <= lo < hi < GROUP_SLOTS):
        raise ValueError(f"malformed nibble 0x{nibble:x}: slot pair ({lo}, {hi}) not strictly increasing")
    return lo, hi


def kept_elements(nibble: int, mode: SparsityMode) -> tuple[int, ...]:
    """codec.py:88-95."""
    lo, hi = slots_for_nibble(nibble)
    if nibble not in mode.admissible_nibbles:
        raise ValueError(f"malformed nibble 0x{nibble:x} for mode {mode.value}")
    if mode is SparsityMode.ONE_OF_TWO:
        return (lo // 2,)
    return (lo, hi)


class GroupSelection(NamedTuple):
    kept: tuple[int, ...]
    slots: tuple[int, int]
    nibble: int


def select_group(values, mode: SparsityMode, device=None) -> GroupSelection:
    """codec.py:104-123, evaluated by the device selection routine itself."""
    mode = as_mode(mode)
    # the reference compares in float64 (codec.py:111); a 16/32-bit tensor is compared as fp32 by
    # the epilogue's own routine (select24 / select12), anything else in float64
    vals = values if isinstance(values, torch.Tensor) else torch.from_numpy(np.asarray(values, dtype=np.float64))
    vals = vals.to(torch.float64 if vals.dtype == torch.float64 else torch.float32).reshape(-1)
    if vals.shape != (mode.group_size,):
        raise ValueError(
            f"expected a group of {mode.group_size} values for mode {mode.value}, got shape {tuple(vals.shape)}"
        )
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    _, meta, _ = _prune(vals.to(dev).reshape(1, -1), mode, vals.dtype, want_kept=False)
    nib = int(meta.item())
    lo, hi = slots_for_nibble(nib)
    return GroupSelection(kept_elements(nib, mode), (lo, hi), nib)


@dataclass(frozen=True, eq=False)
class PruneMask:
    """Boolean keep-mask with exactly N true entries per M-group per row (codec.py:126-147)."""

    bits: torch.Tensor

    def __post_init__(self) -> None:
        if self.bits.dim() < 2:
            raise ValueError("mask must be 2-D")

    @property
    def rows(self) -> int:
        return self.bits.shape[-2]

    @property
    def cols(self) -> int:
        return self.bits.shape[-1]

    def density(self) -> float:
        return float(self.bits.float().mean())


@dataclass(frozen=True, eq=False)
class BlockMask:
    """Tile-grid keep mask for hybrid blocked-ELL sparsity (codec.py:150-200).

    ``keep`` is a host boolean grid shared by every (batch, head); the device
    copy handed to the kernels is cached per device.
    """

    keep: np.ndarray
    tile_rows: int = 32
    tile_cols: int = 64

    def __post_init__(self) -> None:
        keep = self.keep.cpu().numpy() if isinstance(self.keep, torch.Tensor) else self.keep
        arr = np.ascontiguousarray(keep, dtype=bool)
        if arr.ndim != 2:
            raise ValueError("block mask grid must be 2-D")
        if self.tile_rows < 1 or self.tile_cols < 1:
            raise ValueError("tile dimensions must be >= 1")
        object.__setattr__(self, "keep", arr)
        object.__setattr__(self, "_dev", {})

    @property
    def grid_rows(self) -> int:
        return self.keep.shape[0]

    @property
    def grid_cols(self) -> int:
        return self.keep.shape[1]

    def check_covers(self, rows: int, cols: int) -> None:
        want = (-(-rows // self.tile_rows), -(-cols // self.tile_cols))
        if (self.grid_rows, self.grid_cols) != want:
            raise ValueError(
                f"block mask grid {self.keep.shape} does not match the "
                f"{want[0]}x{want[1]} tile grid of a {rows}x{cols} matrix"
            )

    def dense_keep(self, rows: int, cols: int) -> np.ndarray:
        self.check_covers(rows, cols)
        out = np.repeat(np.repeat(self.keep, self.tile_rows, 0), self.tile_cols, 1)
        return np.ascontiguousarray(out[:rows, :cols])

    def nonzero_keep(self, rows: int, dense_cols: int) -> np.ndarray:
        if self.tile_cols % 2:
            raise ValueError("tile_cols must be even to map tiles onto nonzeros")
        self.check_covers(rows, dense_cols)
        out = np.repeat(np.repeat(self.keep, self.tile_rows, 0), self.tile_cols // 2, 1)
        return np.ascontiguousarray(out[:rows, : dense_cols // 2])

    def device_keep(self, device: torch.device) -> torch.Tensor:
        key = str(device)
        if key not in self._dev:
            self._dev[key] = torch.from_numpy(self.keep.astype(np.uint8)).to(device)
        return self._dev[key]


def meta_hw_words(mode: SparsityMode, rows: int, dense_cols: int) -> int:
    """Words of one (batch, head) meta_hw block (include/dfss.h)."""
    return int(_lib.load().dfss_meta_hw_words(mode.group_size, 1, rows, dense_cols))


def _meta_words_host(mode: SparsityMode, rows: int, dense_cols: int) -> int:
    groups = dense_cols // mode.group_size
    return (-(-rows // 128)) * (-(-groups // 8)) * 128


@dataclass(frozen=True, eq=False)
class CompressedSparse:
    """Nonzeros (N/M of dense) plus nibble metadata, on the GPU (codec.py:203-282).

    nonzeros: [..., rows, dense_cols/2]; meta_hw: int32 [..., words] in the
    tcgen05 lane layout.  ``metadata`` gives the reference's LOGICAL nibble
    stream ([..., rows * dense_cols/gs] uint8; zero filler in masked tiles).
    """

    rows: int
    dense_cols: int
    mode: SparsityMode
    nonzeros: torch.Tensor
    meta_hw: torch.Tensor
    layout: Layout = Layout.LOGICAL
    block_mask: BlockMask | None = None
    #: optional [..., rows, 4] fp32 partial row maxima recorded by the tcgen05 SDDMM
    row_max: torch.Tensor | None = None

    def __post_init__(self) -> None:
        if self.rows < 1 or self.dense_cols < 1:
            raise ValueError("rows and dense_cols must be positive")
        if self.dense_cols % self.mode.group_size != 0:
            raise ValueError(
                f"dense_cols={self.dense_cols} not divisible by group size {self.mode.group_size}"
            )
        if tuple(self.nonzeros.shape[-2:]) != (self.rows, self.dense_cols // 2):
            raise ValueError(
                f"nonzeros shape {tuple(self.nonzeros.shape)} != (..., {self.rows}, {self.dense_cols // 2})"
            )
        words = _meta_words_host(self.mode, self.rows, self.dense_cols)
        if self.meta_hw.shape[-1] != words or self.meta_hw.shape[:-1] != self.nonzeros.shape[:-2]:
            raise ValueError(f"metadata holds {tuple(self.meta_hw.shape)} words, expected (..., {words})")
        if self.block_mask is not None:
            if self.layout is not Layout.LOGICAL:
                raise ValueError("block-masked matrices only support the logical layout")
            self.block_mask.check_covers(self.rows, self.dense_cols)

    # ---- geometry
    @property
    def batch_shape(self) -> tuple[int, ...]:
        return tuple(self.nonzeros.shape[:-2])

    @property
    def bh(self) -> int:
        return int(np.prod(self.batch_shape, dtype=np.int64)) if self.batch_shape else 1

    @property
    def nibbles_per_row(self) -> int:
        return self.dense_cols // self.mode.group_size

    @property
    def nonzero_cols(self) -> int:
        return self.dense_cols // 2

    @property
    def device(self) -> torch.device:
        return self.nonzeros.device

    # ---- logical views (parity / interchange; not on the hot path)
    @property
    def metadata(self) -> torch.Tensor:
        """LOGICAL nibble stream, one nibble per byte, [..., rows * groups]."""
        out = torch.empty(self.batch_shape + (self.rows * self.nibbles_per_row,), dtype=torch.uint8,
                          device=self.device)
        lib = _lib.load()
        with torch.cuda.device(self.device):
            _lib.check(lib.dfss_meta_hw_to_logical(_lib.ptr(self.meta_hw), _lib.ptr(out), self.mode.group_size, self.bh,
                                                   self.rows, self.dense_cols, _lib.stream_of(out)), "meta decode")
        if self.block_mask is not None:
            present = self.block_mask.dense_keep(self.rows, self.dense_cols)[:, :: self.mode.group_size]
            out.view(self.batch_shape + (self.rows, self.nibbles_per_row)).mul_(
                torch.from_numpy(present.astype(np.uint8)).to(self.device))
        return out

    def meta_grid(self) -> torch.Tensor:
        if self.layout is not Layout.LOGICAL:
            raise ValueError("metadata grid is only defined for the logical layout")
        return self.metadata.view(self.batch_shape + (self.rows, self.nibbles_per_row))

    def present_nonzeros(self) -> torch.Tensor:
        if self.block_mask is None:
            return torch.ones((self.rows, self.nonzero_cols), dtype=torch.bool, device=self.device)
        return torch.from_numpy(self.block_mask.nonzero_keep(self.rows, self.dense_cols)).to(self.device)

    @classmethod
    def from_logical(cls, rows: int, dense_cols: int, mode: SparsityMode, nonzeros: torch.Tensor,
                     metadata: torch.Tensor, block_mask: BlockMask | None = None) -> "CompressedSparse":
        """Build from the reference's logical stream; validates every nibble (codec.py:248-262)."""
        mode = as_mode(mode)
        _lib.require_cuda(nonzeros)
        groups = dense_cols // mode.group_size
        meta = torch.as_tensor(metadata).to(device=nonzeros.device, dtype=torch.uint8)
        batch = tuple(nonzeros.shape[:-2])
        meta = meta.reshape(batch + (rows * groups,))
        legal = torch.zeros(16, dtype=torch.bool, device=meta.device)
        legal[list(mode.admissible_nibbles)] = True
        bad = ~legal[meta.long()]
        if block_mask is not None:
            present = block_mask.dense_keep(rows, dense_cols)[:, :: mode.group_size].ravel()
            bad &= torch.from_numpy(present).to(meta.device)
        if bool(bad.any()):
            flat = bad.reshape(-1)
            idx = int(torch.nonzero(flat)[0])
            raise ValueError(
                f"malformed nibble 0x{int(meta.reshape(-1)[idx]):x} at position {idx % (rows * groups)} "
                f"for mode {mode.value}"
            )
        if block_mask is not None:
            present = torch.from_numpy(block_mask.dense_keep(rows, dense_cols)[:, :: mode.group_size].ravel())
            meta = torch.where(present.to(meta.device), meta, torch.full_like(meta, 0x4))
        words = _meta_words_host(mode, rows, dense_cols)
        hw = torch.empty(batch + (words,), dtype=torch.int32, device=nonzeros.device)
        bh = int(np.prod(batch, dtype=np.int64)) if batch else 1
        lib = _lib.load()
        with torch.cuda.device(hw.device):
            _lib.check(lib.dfss_meta_logical_to_hw(_lib.ptr(meta.contiguous()), _lib.ptr(hw), mode.group_size, bh, rows,
                                                   dense_cols, _lib.stream_of(hw)), "meta encode")
        return cls(rows, dense_cols, mode, nonzeros.contiguous(), hw, block_mask=block_mask)


# ---------------------------------------------------------------------------
# selection on given scores (the parity hook, codec.py:289-335)


def _prune(scores: torch.Tensor, mode: SparsityMode, nz_dtype: torch.dtype, want_kept: bool = True):
    """Run dfss_prune_scores: (nonzeros, logical meta [rows, groups], kept uint8 [rows, cols]).
    float64 scores are compared in float64 (dfss_prune_scores_f64), never rounded first."""
    _lib.require_cuda(scores)
    if scores.dtype == torch.float64:
        from . import kernels_f64

        if scores.shape[-1] % mode.group_size:
            raise ValueError(f"column count {scores.shape[-1]} not divisible by group size {mode.group_size} "
                             f"(mode {mode.value})")
        nz, meta, kept = kernels_f64.prune_scores(scores, mode.group_size, want_kept)
        return (nz if nz_dtype == torch.float64 else nz.to(nz_dtype)), meta, kept
    s = scores.contiguous().to(torch.float32)
    cols = s.shape[-1]
    rows = s.numel() // cols if cols else 0
    gs = mode.group_size
    if cols % gs:
        raise ValueError(f"column count {cols} not divisible by group size {gs} (mode {mode.value})")
    nz = torch.empty(s.shape[:-1] + (cols // 2,), dtype=nz_dtype, device=s.device)
    meta = torch.empty(s.shape[:-1] + (cols // gs,), dtype=torch.uint8, device=s.device)
    kept = torch.empty(s.shape, dtype=torch.uint8, device=s.device) if want_kept else None
    lib = _lib.load()
    with torch.cuda.device(s.device):
        _lib.check(lib.dfss_prune_scores(_lib.ptr(s), _lib.ptr(nz), _lib.ptr(meta), _lib.ptr(kept), gs,
                                         _lib.dtype_id(nz_dtype), rows, cols, _lib.stream_of(s)), "prune_scores")
    return nz, meta, kept


def prune_scores(scores: torch.Tensor, mode, nz_dtype: torch.dtype = torch.float32):
    """Select on a given fp32 score tensor with the SDDMM epilogue's own routine.

    Returns (nonzeros, logical nibbles [..., rows, groups], kept bool [..., rows, cols]).
    """
    nz, meta, kept = _prune(scores, as_mode(mode), nz_dtype)
    return nz, meta, kept.bool()


def compress_logical(m, mode) -> CompressedSparse:
    """codec.py:331-335 on the device."""
    from .dense import as_tensor

    mode = as_mode(mode)
    data = as_tensor(m)
    if data.shape[-1] % mode.group_size:
        raise ValueError(
            f"column count {data.shape[-1]} not divisible by group size {mode.group_size} (mode {mode.value})"
        )
    nz, meta, _ = _prune(data, mode, data.dtype, want_kept=False)
    return CompressedSparse.from_logical(data.shape[-2], data.shape[-1], mode, nz, meta)


def prune_dense(m, mode):
    """codec.py:324-328 on the device: (pruned dense, PruneMask)."""
    from .dense import DenseMatrix, as_tensor

    mode = as_mode(mode)
    data = as_tensor(m)
    _, _, kept = _prune(data, mode, data.dtype)
    kept = kept.bool()
    return DenseMatrix(torch.where(kept, data, torch.zeros_like(data)), check_finite=False), PruneMask(kept)


def nonzero_columns(c: CompressedSparse) -> torch.Tensor:
    """codec.py:346-360: dense column of every stored nonzero (-1 in masked tiles)."""
    if c.layout is not Layout.LOGICAL:
        raise ValueError("column decode requires the logical layout")
    meta = c.meta_grid().long()
    groups = torch.arange(c.nibbles_per_row, device=c.device, dtype=torch.int64)
    if c.mode is SparsityMode.ONE_OF_TWO:
        cols = 2 * groups + (meta == 0xE).long()
    else:
        base = 4 * groups
        cols = torch.stack((base + (meta & 3), base + ((meta >> 2) & 3)), dim=-1)
        cols = cols.reshape(c.batch_shape + (c.rows, c.nonzero_cols))
    if c.block_mask is not None:
        cols = torch.where(c.present_nonzeros(), cols, torch.full_like(cols, -1))
    return cols.contiguous()


def decompress(c: CompressedSparse):
    """codec.py:363-372: scatter nonzeros back to dense positions (masked tiles stay zero)."""
    from .dense import DenseMatrix

    if c.layout is not Layout.LOGICAL:
        raise ValueError("decompress requires the logical layout (decode tiles first)")
    cols = nonzero_columns(c)
    present = c.present_nonzeros()
    vals = torch.where(present, c.nonzeros, torch.zeros_like(c.nonzeros))
    # masked entries (-1) land in a spare trailing column that is dropped
    out = torch.zeros(c.batch_shape + (c.rows, c.dense_cols + 1), dtype=c.nonzeros.dtype, device=c.device)
    out.scatter_(-1, torch.where(cols < 0, torch.full_like(cols, c.dense_cols), cols), vals)
    return DenseMatrix(out[..., : c.dense_cols].contiguous(), check_finite=False)


def dense_payload_bits(rows: int, cols: int, element_bits: int = 32) -> int:
    """codec.py:448-450."""
    return rows * cols * element_bits


def compressed_payload_bits(c: CompressedSparse, element_bits: int = 32) -> int:
    """codec.py:453-459: nonzeros plus 4-bit nibbles, per (batch, head)."""
    return c.rows * c.nonzero_cols * element_bits + c.rows * c.nibbles_per_row * 4
