"""CPU oracle for the DFSS attention hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy, the algorithm of the reference package
``nmattn`` 0.1.0 (``/root/reference/pkg/src/nmattn``) for the path that the
B200 product replaces: fused SDDMM + N:M prune, compressed-row softmax, and
the compressed SpMM.  It exists so that ``tests/``, ``__graft_entry__.smoke``
and the ``cpu_baseline`` leg of ``bench.py`` can check and time the CUDA
product against the reference semantics on a machine where the reference
itself is absent (the GPU box).  Nothing in ``paper_2203_00091_b200`` may
import it; the product path fails loudly when its CUDA library is missing.

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors produced by the real reference (``tests/golden/make_golden.py``,
run in the build container where ``/root/reference`` is importable), and the
C restatement (``oracle/dfss_oracle.c``) is checked bitwise against both.

All arithmetic is float64, like the reference (``SPEC.md:70``).
"""

from __future__ import annotations

import math

import numpy as np

ONE_OF_TWO = "1:2"
TWO_OF_FOUR = "2:4"

#: admissible nibble sets, codec.py:59-64
ADMISSIBLE = {
    ONE_OF_TWO: frozenset({0x4, 0xE}),
    TWO_OF_FOUR: frozenset({0x4, 0x8, 0x9, 0xC, 0xD, 0xE}),
}


def group_size(mode: str) -> int:
    """codec.py:47-50 -- 2 elements per group under 1:2, 4 under 2:4."""
    if mode not in ADMISSIBLE:
        raise ValueError(f"unknown sparsity mode {mode!r} (expected '1:2' or '2:4')")
    return 2 if mode == ONE_OF_TWO else 4


def nibble_for_slots(lo: int, hi: int) -> int:
    """codec.py:72-76 -- ``lo | hi << 2`` on the 4-slot grid, lo < hi."""
    if not (0 <= lo < hi < 4):
        raise ValueError(f"slot pair ({lo}, {hi}) must be strictly increasing in [0, 4)")
    return lo | (hi << 2)


def slots_for_nibble(nibble: int) -> tuple[int, int]:
    """codec.py:79-85."""
    lo, hi = nibble & 0x3, (nibble >> 2) & 0x3
    if not (0 <= lo < hi < 4):
        raise ValueError(f"malformed nibble 0x{nibble:x}: slot pair ({lo}, {hi}) not strictly increasing")
    return lo, hi


def select_group(values, mode: str) -> tuple[tuple[int, ...], int]:
    """codec.py:104-123 -- (kept element indices, nibble) for one group.

    1:2 keeps element 1 iff v1 > v0; 2:4 keeps the first two entries of a
    stable descending sort (signed value, ties to the lower index).
    """
    vals = np.asarray(values, dtype=np.float64)
    gs = group_size(mode)
    if vals.shape != (gs,):
        raise ValueError(f"expected a group of {gs} values for mode {mode}, got shape {vals.shape}")
    if mode == ONE_OF_TWO:
        kept = 1 if vals[1] > vals[0] else 0
        return (kept,), nibble_for_slots(2 * kept, 2 * kept + 1)
    order = np.argsort(-vals, kind="stable")
    lo, hi = sorted(int(i) for i in order[:2])
    return (lo, hi), nibble_for_slots(lo, hi)


def select_rows(values: np.ndarray, mode: str):
    """codec.py:289-313 -- vectorised selection over a (rows, cols) array.

    Returns (kept bool [rows, cols], nonzeros f64 [rows, cols/2],
    nibbles u8 [rows, cols/gs]).
    """
    values = np.asarray(values, dtype=np.float64)
    rows, cols = values.shape
    gs = group_size(mode)
    if cols % gs:
        raise ValueError(f"column count {cols} not divisible by group size {gs} (mode {mode})")
    grouped = values.reshape(rows, cols // gs, gs)
    if mode == ONE_OF_TWO:
        second = grouped[:, :, 1] > grouped[:, :, 0]
        kept = np.zeros(grouped.shape, dtype=bool)
        kept[:, :, 0] = ~second
        kept[:, :, 1] = second
        nonzeros = np.where(second, grouped[:, :, 1], grouped[:, :, 0])
        nibbles = np.where(second, 0xE, 0x4).astype(np.uint8)
        return kept.reshape(rows, cols), nonzeros, nibbles
    order = np.argsort(-grouped, axis=2, kind="stable")
    top2 = np.sort(order[:, :, :2], axis=2)
    kept = np.zeros(grouped.shape, dtype=bool)
    np.put_along_axis(kept, top2, True, axis=2)
    nonzeros = np.take_along_axis(grouped, top2, axis=2).reshape(rows, cols // 2)
    nibbles = (top2[:, :, 0] | (top2[:, :, 1] << 2)).astype(np.uint8)
    return kept.reshape(rows, cols), nonzeros, nibbles


def compress_logical(scores: np.ndarray, mode: str):
    """codec.py:331-335 -- (nonzeros [r, c/2], flat logical nibbles [r*c/gs])."""
    _, nz, nib = select_rows(scores, mode)
    return nz, nib.ravel()


def prune_dense(scores: np.ndarray, mode: str):
    """codec.py:324-328 -- (pruned dense, kept mask)."""
    kept, _, _ = select_rows(scores, mode)
    return np.where(kept, scores, 0.0), kept


def nonzero_columns(meta: np.ndarray, rows: int, dense_cols: int, mode: str) -> np.ndarray:
    """codec.py:346-360 -- dense column index of each stored nonzero."""
    gs = group_size(mode)
    grid = np.asarray(meta, dtype=np.int64).reshape(rows, dense_cols // gs)
    groups = np.arange(dense_cols // gs, dtype=np.int64)
    if mode == ONE_OF_TWO:
        return 2 * groups[None, :] + (grid == 0xE)
    lo = grid & 0x3
    hi = (grid >> 2) & 0x3
    base = 4 * groups[None, :]
    return np.stack((base + lo, base + hi), axis=2).reshape(rows, dense_cols // 2)


def decompress(nonzeros: np.ndarray, meta: np.ndarray, dense_cols: int, mode: str) -> np.ndarray:
    """codec.py:363-372 -- scatter nonzeros back to dense positions."""
    rows = nonzeros.shape[0]
    cols = nonzero_columns(meta, rows, dense_cols, mode)
    out = np.zeros((rows, dense_cols))
    r = np.repeat(np.arange(rows), nonzeros.shape[1])
    out[r, cols.ravel()] = nonzeros.ravel()
    return out


def gemm_scaled(a: np.ndarray, b: np.ndarray, scale: float) -> np.ndarray:
    """dense.py:80-104 / _kernels_numba.py:16-36 -- ``scale * (a @ b.T)``.

    The reference accumulates every element in ascending k into one
    accumulator and multiplies by ``scale`` once at the end; the loop over k
    below reproduces that order exactly (numpy's matmul does not guarantee
    it), so results are bitwise equal to the reference.
    """
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    acc = np.zeros((a.shape[0], b.shape[0]))
    for k in range(a.shape[1]):
        acc += a[:, k : k + 1] * b[None, :, k]
    return acc * scale


def sddmm_compress(q: np.ndarray, k: np.ndarray, scale: float, mode: str):
    """_kernels_numba.py:110-185 (no block mask) -- fused score + prune.

    Tile traversal does not change any element's value (ascending-k single
    accumulator, scale applied once), so the fused result equals
    ``compress_logical(gemm_scaled(q, k, scale))`` bitwise (test_fused.py:30-43).
    """
    return compress_logical(gemm_scaled(q, k, scale), mode)


def softmax_nonzeros(nz: np.ndarray, present: np.ndarray | None = None) -> np.ndarray:
    """_kernels_numba.py:66-84 -- three passes: max, exp + sequential sum, divide."""
    nz = np.asarray(nz, dtype=np.float64)
    if present is None:
        present = np.ones(nz.shape, dtype=bool)
    masked = np.where(present, nz, -np.inf)
    mx = masked.max(axis=1, keepdims=True)
    e = np.where(present, np.exp(nz - mx), 0.0)
    # the reference sums sequentially in ascending column order
    s = np.zeros((nz.shape[0], 1))
    for j in range(nz.shape[1]):
        s[:, 0] += e[:, j]
    return np.where(present, e / s, 0.0)


def spmm_gather(nz: np.ndarray, cols: np.ndarray, v: np.ndarray, present: np.ndarray | None = None) -> np.ndarray:
    """_kernels_numba.py:91-103 -- ``out[i,:] += nz[i,c] * v[cols[i,c],:]`` in ascending c."""
    nz = np.asarray(nz, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    if present is None:
        present = np.ones(nz.shape, dtype=bool)
    out = np.zeros((nz.shape[0], v.shape[1]))
    for c in range(nz.shape[1]):
        contrib = nz[:, c : c + 1] * v[cols[:, c]]
        out += np.where(present[:, c : c + 1], contrib, 0.0)
    return out


def nm_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, mode: str) -> np.ndarray:
    """pipeline.py:15-32 -- attention_sddmm -> softmax_rows -> spmm, scale 1/sqrt(d) (fused.py:110)."""
    n, d = q.shape
    nz, meta = sddmm_compress(q, k, 1.0 / math.sqrt(d), mode)
    p = softmax_nonzeros(nz)
    cols = nonzero_columns(meta, n, k.shape[0], mode)
    return spmm_gather(p, cols, v)


def full_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray) -> np.ndarray:
    """dense.py:118-122 -- softmax(Q K^T / sqrt(d)) V, the CPU dense comparator."""
    s = gemm_scaled(q, k, 1.0 / math.sqrt(q.shape[1]))
    mx = s.max(axis=1, keepdims=True)
    e = np.exp(s - mx)
    acc = np.zeros((s.shape[0], 1))
    for j in range(s.shape[1]):
        acc[:, 0] += e[:, j]
    w = e / acc
    return gemm_scaled(w, np.ascontiguousarray(np.asarray(v, dtype=np.float64).T), 1.0)


def approx_error(full: np.ndarray, sparse: np.ndarray):
    """pipeline.py:49-57 -- (rel_l2, max_abs, per-row relative l2)."""
    if full.shape != sparse.shape:
        raise ValueError(f"shape mismatch: {full.shape} vs {sparse.shape}")
    diff = full - sparse
    denom = np.linalg.norm(full)
    rel = float(np.linalg.norm(diff) / denom) if denom > 0 else 0.0
    row_norms = np.linalg.norm(full, axis=1)
    safe = np.where(row_norms > 0, row_norms, 1.0)
    row_rel = np.where(row_norms > 0, np.linalg.norm(diff, axis=1) / safe, 0.0)
    return rel, float(np.abs(diff).max()), row_rel
