"""Dense containers and the dense attention baseline on the GPU (reference: dense.py).

``DenseMatrix`` / ``AttentionInputs`` keep the reference's names and checks
(dense.py:19-77) over CUDA tensors with optional leading batch dimensions.
The dense baseline (``gemm_scaled``, ``full_attention``, dense.py:80-122) is
the cuBLAS comparator the paper measures against for 16/32-bit data; on
float64 data (the reference's dtype) it runs the reference's own arithmetic
(kernels_f64: ascending single-accumulator GEMM, sequential softmax sums), so
it returns the reference's numbers.  Dtypes are never narrowed silently:
float64 stays float64.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch


def _to_device_tensor(data) -> torch.Tensor:
    if isinstance(data, DenseMatrix):
        return data.data
    if isinstance(data, torch.Tensor):
        t = data
    else:
        t = torch.as_tensor(np.asarray(data))
    if t.dtype not in (torch.float64, torch.float32, torch.bfloat16, torch.float16):
        t = t.to(torch.float64 if not t.is_floating_point() else torch.float32)
    if not t.is_cuda:
        if not torch.cuda.is_available():
            return t  # shape validation still works; kernels will refuse CPU tensors
        t = t.cuda()
    return t


def as_tensor(x) -> torch.Tensor:
    return _to_device_tensor(x)


@dataclass(frozen=True, eq=False)
class DenseMatrix:
    """Row-major [..., rows, cols] matrix on the GPU; finite entries only (dense.py:19-52)."""

    data: torch.Tensor
    check_finite: bool = True

    def __post_init__(self) -> None:
        t = _to_device_tensor(self.data)
        if t.dim() < 2:
            raise ValueError(f"expected a 2-D matrix, got {t.dim()}-D")
        if t.shape[-2] < 1 or t.shape[-1] < 1:
            raise ValueError(f"matrix dimensions must be positive, got {tuple(t.shape)}")
        if self.check_finite and not bool(torch.isfinite(t).all()):
            raise ValueError("matrix entries must be finite (no NaN/Inf)")
        object.__setattr__(self, "data", t.contiguous())

    @property
    def rows(self) -> int:
        return self.data.shape[-2]

    @property
    def cols(self) -> int:
        return self.data.shape[-1]

    @property
    def shape(self) -> tuple[int, ...]:
        return tuple(self.data.shape)

    @classmethod
    def zeros(cls, rows: int, cols: int, dtype=torch.float32) -> "DenseMatrix":
        return cls(torch.zeros((rows, cols), dtype=dtype, device="cuda"))


@dataclass(frozen=True)
class AttentionInputs:
    """Query/key/value sharing (…, n, d) (dense.py:55-77)."""

    q: DenseMatrix
    k: DenseMatrix
    v: DenseMatrix

    def __post_init__(self) -> None:
        for name in ("q", "k", "v"):
            val = getattr(self, name)
            if not isinstance(val, DenseMatrix):
                object.__setattr__(self, name, DenseMatrix(val))
        shape = self.q.shape
        if self.k.shape != shape or self.v.shape != shape:
            raise ValueError(
                f"Q, K, V must share shape (n, d); got {self.q.shape}, {self.k.shape}, {self.v.shape}"
            )

    @property
    def n(self) -> int:
        return self.q.rows

    @property
    def d(self) -> int:
        return self.q.cols


def gemm_scaled(a, b, scale: float, **_tiling) -> DenseMatrix:
    """``scale * a @ b^T`` (dense.py:80-104): float64 with the reference's ascending single
    accumulator (bitwise the reference), otherwise cuBLAS with fp32 accumulation."""
    a, b = as_tensor(a), as_tensor(b)
    if a.shape[-1] != b.shape[-1]:
        raise ValueError(f"shape mismatch: inner dims differ ({a.shape[-1]} vs {b.shape[-1]})")
    if a.dtype == torch.float64 or b.dtype == torch.float64:
        from . import kernels_f64

        a64, b64 = a.to(torch.float64), b.to(torch.float64)
        if a64.shape[:-2] != b64.shape[:-2]:
            raise ValueError(f"shape mismatch: batch dims {tuple(a64.shape[:-2])} vs {tuple(b64.shape[:-2])}")
        out = kernels_f64.batched(lambda x, y: kernels_f64.gemm_abt(x, y, scale), a64, b64)
        return DenseMatrix(out, check_finite=False)
    return DenseMatrix(torch.matmul(a, b.transpose(-1, -2)) * scale, check_finite=False)


def attention_scores(inputs: AttentionInputs) -> DenseMatrix:
    return gemm_scaled(inputs.q, inputs.k, 1.0 / math.sqrt(inputs.d))


def dense_attention_weights(inputs: AttentionInputs) -> DenseMatrix:
    s = attention_scores(inputs).data
    if s.dtype == torch.float64:  # _kernels_numba.row_softmax_dense arithmetic
        from . import kernels_f64

        return DenseMatrix(kernels_f64.row_softmax_dense(s), check_finite=False)
    return DenseMatrix(torch.softmax(s.float(), dim=-1).to(s.dtype), check_finite=False)


def full_attention(inputs: AttentionInputs) -> DenseMatrix:
    """Unfused dense baseline softmax(QK^T/sqrt d) V (dense.py:118-122): cuBLAS -> softmax -> cuBLAS."""
    w = dense_attention_weights(inputs).data
    if w.dtype == torch.float64:  # gemm_scaled(weights, V^T, 1.0) as the reference (dense.py:118-122)
        return gemm_scaled(w, inputs.v.data.to(torch.float64).transpose(-1, -2).contiguous(), 1.0)
    return DenseMatrix(torch.matmul(w, inputs.v.data), check_finite=False)
