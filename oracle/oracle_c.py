"""ctypes wrapper for oracle/liboracle_dfss.so -- TEST INFRASTRUCTURE ONLY.

The C restatement (dfss_oracle.c) of the reference numba kernels, used by
tests/ as a bitwise checker and by bench.py as the timed CPU baseline.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle_dfss.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i64 = ctypes.c_int64


def build() -> str:
    """Compile the oracle with its Makefile (no-op when up to date)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "dfss_oracle.c")
        ):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.oracle_sddmm_compress.argtypes = [_dp, _dp, _i64, _i64, _i64, ctypes.c_double, ctypes.c_int,
                                               ctypes.c_int, ctypes.c_int, _u8p, _dp, _u8p, _i64p]
        _lib.oracle_softmax_nonzeros.argtypes = [_dp, _u8p, _i64, _i64, _dp]
        _lib.oracle_spmm_gather.argtypes = [_dp, _i64p, _u8p, _i64, _i64, _dp, _i64, _dp]
        _lib.oracle_nonzero_columns.argtypes = [_u8p, _i64, _i64, ctypes.c_int, _i64p]
        _lib.oracle_gemm_abt.argtypes = [_dp, _dp, _i64, _i64, _i64, ctypes.c_double, _dp]
        _lib.oracle_nm_attention.argtypes = [_dp, _dp, _dp, _i64, _i64, ctypes.c_int, _dp]
        _lib.oracle_full_attention.argtypes = [_dp, _dp, _dp, _i64, _i64, _dp]
        _lib.oracle_attention_batched.argtypes = [_dp, _dp, _dp, _i64, _i64, _i64, ctypes.c_int,
                                                  ctypes.c_int, ctypes.c_int, _dp]
        _lib.oracle_attention_batched.restype = ctypes.c_int
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def _gs(mode: str) -> int:
    return 2 if mode == "1:2" else 4


def sddmm_compress(q, k, scale, mode, tile_rows=32, tile_cols=64, keep=None):
    """_kernels_numba.py:110-185.  Returns (nonzeros, meta [n, m/gs], (peak, nnz, nib))."""
    q, k = _f64(q), _f64(k)
    n, d = q.shape
    m = k.shape[0]
    gs = _gs(mode)
    nz = np.empty((n, m // 2))
    meta = np.empty((n, m // gs), dtype=np.uint8)
    stats = np.zeros(3, dtype=np.int64)
    kp = None if keep is None else np.ascontiguousarray(keep, dtype=np.uint8)
    lib().oracle_sddmm_compress(_ptr(q, _dp), _ptr(k, _dp), n, m, d, float(scale), gs, tile_rows,
                                tile_cols, _ptr(kp, _u8p), _ptr(nz, _dp), _ptr(meta, _u8p),
                                _ptr(stats, _i64p))
    return nz, meta, tuple(int(x) for x in stats)


def softmax_nonzeros(nz, present=None):
    nz = _f64(nz)
    out = np.empty_like(nz)
    p = None if present is None else np.ascontiguousarray(present, dtype=np.uint8)
    lib().oracle_softmax_nonzeros(_ptr(nz, _dp), _ptr(p, _u8p), nz.shape[0], nz.shape[1], _ptr(out, _dp))
    return out


def nonzero_columns(meta, rows, dense_cols, mode):
    meta = np.ascontiguousarray(meta, dtype=np.uint8).ravel()
    cols = np.empty((rows, dense_cols // 2), dtype=np.int64)
    lib().oracle_nonzero_columns(_ptr(meta, _u8p), rows, dense_cols, _gs(mode), _ptr(cols, _i64p))
    return cols


def spmm_gather(nz, cols, v, present=None):
    nz, v = _f64(nz), _f64(v)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    p = None if present is None else np.ascontiguousarray(present, dtype=np.uint8)
    out = np.empty((nz.shape[0], v.shape[1]))
    lib().oracle_spmm_gather(_ptr(nz, _dp), _ptr(cols, _i64p), _ptr(p, _u8p), nz.shape[0], nz.shape[1],
                             _ptr(v, _dp), v.shape[1], _ptr(out, _dp))
    return out


def gemm_scaled(a, b, scale):
    a, b = _f64(a), _f64(b)
    out = np.empty((a.shape[0], b.shape[0]))
    lib().oracle_gemm_abt(_ptr(a, _dp), _ptr(b, _dp), a.shape[0], b.shape[0], a.shape[1], float(scale),
                          _ptr(out, _dp))
    return out


def nm_attention(q, k, v, mode):
    q, k, v = _f64(q), _f64(k), _f64(v)
    out = np.empty_like(q)
    lib().oracle_nm_attention(_ptr(q, _dp), _ptr(k, _dp), _ptr(v, _dp), q.shape[0], q.shape[1], _gs(mode),
                              _ptr(out, _dp))
    return out


def full_attention(q, k, v):
    q, k, v = _f64(q), _f64(k), _f64(v)
    out = np.empty_like(q)
    lib().oracle_full_attention(_ptr(q, _dp), _ptr(k, _dp), _ptr(v, _dp), q.shape[0], q.shape[1],
                                _ptr(out, _dp))
    return out


def attention_batched(q, k, v, mode, nthreads, dense=False):
    """q,k,v: [bh, n, d] -> [bh, n, d]; heads split across ``nthreads`` pthreads."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    bh, n, d = q.shape
    out = np.empty_like(q)
    lib().oracle_attention_batched(_ptr(q, _dp), _ptr(k, _dp), _ptr(v, _dp), bh, n, d, _gs(mode),
                                   int(dense), int(nthreads), _ptr(out, _dp))
    return out
