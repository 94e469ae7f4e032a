"""torch.nn.Module wrapper: DFSS attention as a drop-in for a model's score/softmax/PV block."""

from __future__ import annotations

import torch

from .codec import as_mode
from .pipeline import dfss_attention


class DFSSAttention(torch.nn.Module):
    """softmax over the N:M-pruned scores, times V, for [B, H, n, d] q/k/v (inference)."""

    def __init__(self, mode: str = "2:4", math_mode: str = "auto"):
        super().__init__()
        self.mode = as_mode(mode)
        self.math_mode = math_mode

    def forward(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
        return dfss_attention(q, k, v, self.mode, math_mode=self.math_mode)

    def extra_repr(self) -> str:
        return f"mode={self.mode.value}, math={self.math_mode}"
