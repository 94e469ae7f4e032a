"""ctypes binding to libdfss_sm100a.so (the C ABI in include/dfss.h).

This is the only place the product touches native code.  There is no CPU
or Python fallback: if the library is missing or cannot load, every entry
point raises.  Status codes map to the reference's exception types --
validation failures to ``ValueError`` (the reference validates in its
wrappers, fused.py:58-82), CUDA failures to ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# DFSS_LIB: an alternative build of the same library (kernel experiments in tools/)
LIB_PATH = os.environ.get("DFSS_LIB") or os.path.join(_HERE, "lib", "libdfss_sm100a.so")

DFSS_OK, DFSS_ERR_INVALID, DFSS_ERR_UNSUPPORTED, DFSS_ERR_CUDA, DFSS_ERR_NO_DEVICE = 0, -1, -2, -3, -4
F32, BF16, F16 = 0, 1, 2
MATH_AUTO, MATH_FFMA, MATH_TF32 = 0, 1, 2

DTYPE_ID = {torch.float32: F32, torch.bfloat16: BF16, torch.float16: F16}

_vp = ctypes.c_void_p
_i32 = ctypes.c_int
_i64 = ctypes.c_int64
_f32 = ctypes.c_float

#: exported symbol -> (restype, argtypes); must match include/dfss.h exactly
SIGNATURES = {
    "dfss_meta_hw_words": (_i64, [_i32, _i64, _i64, _i64]),
    "dfss_sddmm_prune": (_i32, [_vp, _vp, _vp, _vp, _f32, _i32, _i32, _i32, _i32, _i64, _i32, _i32, _i32, _vp, _i32,
                                _i32, _vp, _vp, _vp]),
    "dfss_softmax_rows": (_i32, [_vp, _vp, _i32, _i32, _i64, _i32, _i32, _vp, _i32, _i32, _vp, _vp]),
    "dfss_spmm": (_i32, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i64, _i32, _i32, _i32, _vp, _i32, _i32, _vp,
                         _vp]),
    "dfss_nm_attention_workspace_bytes": (_i64, [_i32, _i32, _i64, _i32, _i32]),
    "dfss_nm_attention_workspace_bytes_for": (_i64, [_i32, _i32, _i32, _i64, _i32, _i32, _i32, _i32, _i32]),
    "dfss_nm_attention": (_i32, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i64, _i32, _i32, _vp, _i64, _vp]),
    "dfss_nm_attention_masked": (_i32, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i64, _i32, _i32, _vp, _i32, _i32, _vp,
                                        _i64, _vp]),
    "dfss_nm_attention_dump": (_i32, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i64, _i32, _i32, _vp, _i32, _i32, _vp,
                                      _i64, _vp, _vp, _vp, _vp]),
    "dfss_nm_attention_path": (_i32, [_i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32]),
    "dfss_nm_attention_path_bh": (_i32, [_i32, _i32, _i32, _i64, _i32, _i32, _i32, _i32, _i32]),
    "dfss_prune_scores": (_i32, [_vp, _vp, _vp, _vp, _i32, _i32, _i64, _i32, _vp]),
    "dfss_prune_scores_f64": (_i32, [_vp, _vp, _vp, _vp, _i32, _i64, _i32, _vp]),
    "dfss_meta_hw_to_logical": (_i32, [_vp, _vp, _i32, _i64, _i32, _i32, _vp]),
    "dfss_meta_logical_to_hw": (_i32, [_vp, _vp, _i32, _i64, _i32, _i32, _vp]),
    "dfss_kmod_sddmm_compress": (_i32, [_vp, _vp, ctypes.c_double, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp,
                                        _vp]),
    "dfss_kmod_softmax_nonzeros": (_i32, [_vp, _vp, _vp, _i64, _i32, _vp]),
    "dfss_kmod_spmm_gather": (_i32, [_vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp]),
    "dfss_kmod_gemm_abt": (_i32, [_vp, _vp, ctypes.c_double, _i64, _i64, _i32, _vp, _vp]),
    "dfss_kmod_row_softmax_dense": (_i32, [_vp, _vp, _i64, _i32, _vp]),
    "dfss_status_string": (ctypes.c_char_p, [_i32]),
    "dfss_last_error": (ctypes.c_char_p, []),
    "dfss_has_tcgen05": (_i32, []),
    "dfss_version": (_i32, []),
}

_lib = None


class DFSSLibraryMissing(RuntimeError):
    """The sm_100a library is not built; the product has no fallback path."""


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DFSSLibraryMissing(
                f"{LIB_PATH} is missing: build it with `python -m paper_2203_00091_b200.build` "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status: int, what: str) -> None:
    if status == DFSS_OK:
        return
    lib = load()
    detail = lib.dfss_last_error().decode(errors="replace")
    msg = f"{what}: {lib.dfss_status_string(status).decode()} ({detail})"
    if status == DFSS_ERR_INVALID:
        raise ValueError(msg)
    raise RuntimeError(msg)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def stream_of(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def dtype_id(dtype: torch.dtype) -> int:
    try:
        return DTYPE_ID[dtype]
    except KeyError:
        raise ValueError(f"unsupported dtype {dtype}; expected float32, bfloat16 or float16") from None


def require_cuda(*tensors: torch.Tensor) -> None:
    for t in tensors:
        if t is not None and not t.is_cuda:
            raise ValueError("DFSS tensors must live on a CUDA device (B200); there is no CPU path")
