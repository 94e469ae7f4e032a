"""Dense containers and the dense attention baseline on the GPU (reference: dense.py).

``DenseMatrix`` / ``AttentionInputs`` keep the reference's names and checks
(dense.py:19-77) over CUDA tensors with optional leading batch dimensions.
The dense baseline (``gemm_scaled``, ``full_attention``, dense.py:80-122) is
the cuBLAS comparator the paper measures against: it is a measurement
baseline, not part of the DFSS path.
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
    if t.dtype == torch.float64:
        # B200 has no fast FP64; fp64 inputs run on the exact-FP32 path (tolerance 1e-5)
        t = t.to(torch.float32)
    elif t.dtype not in (torch.float32, torch.bfloat16, torch.float16):
        t = t.to(torch.float32)
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
    """``scale * a @ b^T`` on cuBLAS (dense.py:80-104); fp32 accumulate."""
    a, b = as_tensor(a), as_tensor(b)
    if a.shape[-1] != b.shape[-1]:
        raise ValueError(f"shape mismatch: inner dims differ ({a.shape[-1]} vs {b.shape[-1]})")
    return DenseMatrix(torch.matmul(a, b.transpose(-1, -2)) * scale, check_finite=False)


def attention_scores(inputs: AttentionInputs) -> DenseMatrix:
    return gemm_scaled(inputs.q, inputs.k, 1.0 / math.sqrt(inputs.d))


def dense_attention_weights(inputs: AttentionInputs) -> DenseMatrix:
    s = attention_scores(inputs).data
    return DenseMatrix(torch.softmax(s.float(), dim=-1).to(s.dtype), check_finite=False)


def full_attention(inputs: AttentionInputs) -> DenseMatrix:
    """Unfused dense baseline softmax(QK^T/sqrt d) V (dense.py:118-122): cuBLAS -> softmax -> cuBLAS."""
    w = dense_attention_weights(inputs).data
    return DenseMatrix(torch.matmul(w, inputs.v.data), check_finite=False)
