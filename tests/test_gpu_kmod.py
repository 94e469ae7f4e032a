"""The reference kernel module on the GPU (integration/_kernels_cuda.py, include/dfss.h dfss_kmod_*).

The reference's plugin interface is the duck-typed module behind backend.kernels()
(backend.py:63-67): five functions with fixed signatures and return tuples
(_kernels_numba.py:39,62,87,106,188).  integration/_kernels_cuda.py implements them on the B200 in
float64 with the reference's accumulation order.  Fed the golden inputs the REAL reference
recorded (tests/golden/make_golden.py), it must return the reference's outputs: bitwise for
sddmm_compress (nonzeros, metadata, counters), spmm_gather and gemm_abt; within a few ulp for the
two softmaxes (exp is the only difference).  Composing the five functions the way the reference's
wrappers do reproduces nm_attention / full_attention and REL_L2_PIN (test_acceptance.py:49).
"""

from __future__ import annotations

import importlib.util
import math
import os

import numpy as np
import pytest

from conftest import ROOT, golden
from oracle import nmattn_oracle as ref
from oracle import oracle_c

pytestmark = pytest.mark.gpu

REL_L2_PIN = 0.39969464809566535


@pytest.fixture(scope="module")
def kmod():
    spec = importlib.util.spec_from_file_location("_kernels_cuda", os.path.join(ROOT, "integration", "_kernels_cuda.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _ulp_close(got, want, ulps=8):
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape and got.dtype == want.dtype == np.float64
    tol = ulps * np.spacing(np.maximum(np.abs(want), np.finfo(np.float64).tiny))
    bad = np.abs(got - want) > tol
    assert not bad.any(), f"{int(bad.sum())} entries beyond {ulps} ulp; worst {np.abs(got - want).max():.3e}"


def test_sddmm_compress_bitwise_on_reference_cases(kmod):
    g = golden("fused.npz")
    eye = np.eye(4)
    nz, meta, peak, nnz, nib = kmod.sddmm_compress(eye, eye, 1.0, 2, 32, 64, np.ones((1, 1), dtype=bool))
    assert np.array_equal(nz, g["identity_nonzeros"]) and np.array_equal(meta.ravel(), g["identity_metadata"])
    assert [peak, nnz, nib] == g["identity_stats"].tolist()
    for i in range(int(g["n_cases"])):
        mode = str(g[f"case{i}_mode"])
        gs = 2 if mode == "1:2" else 4
        q, k = g[f"case{i}_q"], g[f"case{i}_k"]
        keep = np.ones((-(-q.shape[0] // 32), -(-k.shape[0] // 64)), dtype=bool)
        nz, meta, peak, nnz, nib = kmod.sddmm_compress(q, k, float(g[f"case{i}_scale"]), gs, 32, 64, keep)
        assert nz.dtype == np.float64 and meta.dtype == np.uint8
        assert np.array_equal(nz, g[f"case{i}_nonzeros"]), f"case {i} nonzeros"
        assert np.array_equal(meta.ravel(), g[f"case{i}_metadata"]), f"case {i} metadata"
        assert [peak, nnz, nib] == g[f"case{i}_stats"].tolist(), f"case {i} counters"
    # block-masked (test_fused.py:66-82): masked tiles absent, zero nonzeros and metadata
    nz, meta, peak, nnz, nib = kmod.sddmm_compress(g["masked_q"], g["masked_k"], 1.0, 2, 32, 32, g["masked_keep"])
    assert np.array_equal(nz, g["masked_nonzeros"]) and np.array_equal(meta.ravel(), g["masked_metadata"])
    assert [peak, nnz, nib] == g["masked_stats"].tolist()


def test_softmax_and_spmm_gather_on_reference_cases(kmod):
    g = golden("sparse_ops.npz")
    for i in range(int(g["n_cases"])):
        mode = str(g[f"case{i}_mode"])
        nz = g[f"case{i}_nonzeros"]
        rows, cols = nz.shape[0], int(g[f"case{i}_dense_cols"])
        present = np.ones(nz.shape, dtype=bool)
        _ulp_close(kmod.softmax_nonzeros(nz, present), g[f"case{i}_softmax"])
        colidx = ref.nonzero_columns(g[f"case{i}_metadata"], rows, cols, mode)
        # fed the reference's softmax output, the gather is bitwise the reference's spmm
        out = kmod.spmm_gather(g[f"case{i}_softmax"], colidx, present, g[f"case{i}_v"])
        assert np.array_equal(out, g[f"case{i}_spmm"]), f"case {i} spmm"


def test_arbitrary_present_masks_and_decoded_columns(kmod):
    """The reference kernels take any per-nonzero `present` mask and any decoded columns
    (_kernels_numba.py:66-106); checked against the C restatement (bitwise numba)."""
    rng = np.random.default_rng(11)
    for rows, nzc, m, d in [(37, 24, 48, 19), (128, 256, 512, 64), (5, 3, 6, 1)]:
        nz = rng.standard_normal((rows, nzc)) * 4
        present = rng.random((rows, nzc)) < 0.7
        present[0] = False  # an empty row: all zeros, no division (sparse_ops rejects it before the kernel)
        cols = rng.integers(0, m, size=(rows, nzc)).astype(np.int64)
        v = rng.standard_normal((m, d))
        sm = kmod.softmax_nonzeros(nz, present)
        _ulp_close(sm, oracle_c.softmax_nonzeros(nz, present))
        assert (sm[~present] == 0).all()
        assert np.array_equal(kmod.spmm_gather(sm, cols, present, v), oracle_c.spmm_gather(sm, cols, v, present))
    with pytest.raises(IndexError, match="out of range"):
        kmod.spmm_gather(np.ones((2, 2)), np.array([[0, 9], [1, 0]], dtype=np.int64), np.ones((2, 2), bool),
                         np.ones((4, 3)))


def _nm_attention_via_kmod(kmod, q, k, v, mode):
    """pipeline.nm_attention (pipeline.py:15-32) composed from the kernel module like the reference
    wrappers: sddmm_prune (fused.py:41-96) -> softmax_rows (sparse_ops.py:18-37) -> spmm (:40-68)."""
    n, d = q.shape
    gs = 2 if mode == "1:2" else 4
    keep = np.ones((-(-n // 32), -(-n // 64)), dtype=bool)
    nz, meta, *_ = kmod.sddmm_compress(q, k, 1.0 / math.sqrt(d), gs, 32, 64, keep)
    present = np.ones(nz.shape, dtype=bool)
    sm = kmod.softmax_nonzeros(nz, present)
    return kmod.spmm_gather(sm, ref.nonzero_columns(meta.ravel(), n, n, mode), present, v), meta


def _full_attention_via_kmod(kmod, q, k, v):
    """dense.full_attention (dense.py:118-122): gemm_scaled -> row_softmax_dense -> gemm_scaled(W, V^T)."""
    w = kmod.row_softmax_dense(kmod.gemm_abt(q, k, 1.0 / math.sqrt(q.shape[1]), 64, 64, 32))
    return kmod.gemm_abt(w, np.ascontiguousarray(v.T), 1.0, 64, 64, 32)


def test_pipeline_and_full_attention_through_the_kernel_module(kmod):
    g = golden("pipeline.npz")
    for i in range(int(g["n_cases"])):
        q, k, v = g[f"case{i}_q"], g[f"case{i}_k"], g[f"case{i}_v"]
        scores = kmod.gemm_abt(q, k, 1.0 / math.sqrt(q.shape[1]), 64, 64, 32)
        assert np.array_equal(scores, ref.gemm_scaled(q, k, 1.0 / math.sqrt(q.shape[1])))  # C oracle bitwise
        for mode in ("1:2", "2:4"):
            key = mode.replace(":", "")
            out, meta = _nm_attention_via_kmod(kmod, q, k, v, mode)
            # fused == unfused on the metadata (acceptance c02): sddmm_compress vs compress_logical(gemm)
            assert np.array_equal(meta.ravel(), g[f"case{i}_meta{key}"])
            assert np.array_equal(ref.compress_logical(scores, mode)[1], g[f"case{i}_meta{key}"])
            np.testing.assert_allclose(out, g[f"case{i}_nm{key}"], rtol=1e-13, atol=1e-15)
    q, k, v = g["pin_q"], g["pin_k"], g["pin_v"]
    full = _full_attention_via_kmod(kmod, q, k, v)
    np.testing.assert_allclose(full, g["pin_full"], rtol=1e-13, atol=1e-15)
    nm24, _ = _nm_attention_via_kmod(kmod, q, k, v, "2:4")
    np.testing.assert_allclose(nm24, g["pin_nm24"], rtol=1e-13, atol=1e-15)
    nm12, _ = _nm_attention_via_kmod(kmod, q, k, v, "1:2")
    np.testing.assert_allclose(nm12, g["pin_nm12"], rtol=1e-13, atol=1e-15)
    rel = ref.approx_error(full, nm12)[0]  # test_acceptance.py:244-245 (1:2)
    assert abs(rel - REL_L2_PIN) <= 1e-12 * REL_L2_PIN


def test_package_float64_path_is_the_reference_arithmetic():
    """float64 data through the package's own reference-shaped API (DenseMatrix keeps float64):
    sddmm_prune / compress_logical / prune_dense bitwise, nm_attention / full_attention to the
    reference's numbers (exp rounding aside) -- no silent narrowing to fp32."""
    import torch

    import paper_2203_00091_b200 as dfss

    g = golden("fused.npz")
    for i in range(int(g["n_cases"])):
        mode = str(g[f"case{i}_mode"])
        c, st = dfss.sddmm_prune(dfss.DenseMatrix(g[f"case{i}_q"]), dfss.DenseMatrix(g[f"case{i}_k"]), mode,
                                 float(g[f"case{i}_scale"]))
        assert c.nonzeros.dtype == torch.float64
        assert np.array_equal(c.nonzeros.cpu().numpy(), g[f"case{i}_nonzeros"]), f"case {i}"
        assert np.array_equal(c.metadata.cpu().numpy(), g[f"case{i}_metadata"]), f"case {i}"
        assert [st.peak_tile_elems, st.nonzeros_written, st.nibbles_written] == g[f"case{i}_stats"].tolist()
    cg = golden("codec.npz")
    for i in range(int(cg["n_scores"])):
        s = cg[f"scores{i}"]
        for mode in ("1:2", "2:4"):
            key = mode.replace(":", "")
            c = dfss.compress_logical(dfss.DenseMatrix(s, check_finite=False), mode)
            assert np.array_equal(c.nonzeros.cpu().numpy(), cg[f"scores{i}_{key}_nonzeros"])
            assert np.array_equal(c.metadata.cpu().numpy(), cg[f"scores{i}_{key}_metadata"])
            _, mask = dfss.prune_dense(dfss.DenseMatrix(s, check_finite=False), mode)
            assert np.array_equal(mask.bits.cpu().numpy(), cg[f"scores{i}_{key}_mask"])
    pg = golden("pipeline.npz")
    q, k, v = (dfss.DenseMatrix(pg[f"pin_{c}"]) for c in "qkv")
    inputs = dfss.AttentionInputs(q, k, v)
    full = dfss.full_attention(inputs).data
    assert full.dtype == torch.float64
    np.testing.assert_allclose(full.cpu().numpy(), pg["pin_full"], rtol=1e-13, atol=1e-15)
    for mode in ("1:2", "2:4"):
        out = dfss.nm_attention(inputs, mode).data
        assert out.dtype == torch.float64
        np.testing.assert_allclose(out.cpu().numpy(), pg[f"pin_nm{mode.replace(':', '')}"], rtol=1e-13, atol=1e-15)
    rel = dfss.approx_error(full, dfss.nm_attention(inputs, "1:2")).rel_l2
    assert abs(rel - REL_L2_PIN) <= 1e-12 * REL_L2_PIN
    # explicit narrowing stays available (exact-FP32 kernels, 1e-5)
    fast = dfss.nm_attention(inputs, "1:2", precision="fp32").data
    assert fast.dtype == torch.float64
    np.testing.assert_allclose(fast.cpu().numpy(), pg["pin_nm12"], rtol=1e-4, atol=1e-5)
