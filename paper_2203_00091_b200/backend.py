"""Kernel backend selection (reference: backend.py).

The reference switches between numba and numpy kernel modules
(backend.py:17-67).  This build has exactly one backend -- the sm_100a CUDA
library -- and no fallback: ``set_backend`` accepts only that name.
"""

from __future__ import annotations

from . import _lib

NAME = "cuda-sm100a"


def set_backend(name: str) -> None:
    if name != NAME:
        raise ValueError(f"unknown backend {name!r}; this build has only {NAME!r} (no CPU fallback)")
    _lib.load()


def active_backend() -> str:
    _lib.load()
    return NAME


def kernels():
    """The loaded C-ABI library (the analogue of the reference's kernel module)."""
    return _lib.load()
