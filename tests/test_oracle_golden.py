"""Pin the CPU oracle (oracle/) to golden vectors produced by the real reference.

CPU-only.  These tests are what makes the oracle trustworthy as the checker
for the GPU parity tests: every numpy and C restatement must reproduce the
reference outputs bitwise (selection, metadata, masks, fused SDDMM, SpMM
gather order) or to the last ulp of exp (softmax), see
tests/golden/make_golden.py for how the fixtures were made.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import nmattn_oracle as ref
from oracle import oracle_c

#: test_acceptance.py:49 -- the reference's own frozen regression value
REL_L2_PIN = 0.39969464809566535


def test_select_group_anchors():
    g = golden("codec.npz")
    for i in range(int(g["n_groups"])):
        mode = str(g[f"group{i}_mode"])
        kept, nib = ref.select_group(g[f"group{i}_values"], mode)
        assert list(kept) == list(g[f"group{i}_kept"]), i
        assert nib == int(g[f"group{i}_nibble"]), i


def test_sum_tie_counterexample_keeps_first_and_third():
    # pair sums tie in fp32; the reference keeps (0, 2) -> 0x8
    kept, nib = ref.select_group([1000.0, np.float32(1e-5), np.float32(2e-5), -3.0], "2:4")
    assert kept == (0, 2) and nib == 0x8


@pytest.mark.parametrize("mode", ["1:2", "2:4"])
def test_compress_and_mask_match_reference(mode):
    g = golden("codec.npz")
    tag = mode.replace(":", "")
    for i in range(int(g["n_scores"])):
        s = g[f"scores{i}"]
        nz, meta = ref.compress_logical(s, mode)
        _, mask = ref.prune_dense(s, mode)
        assert np.array_equal(nz, g[f"scores{i}_{tag}_nonzeros"]), i
        assert np.array_equal(meta, g[f"scores{i}_{tag}_metadata"]), i
        assert np.array_equal(mask, g[f"scores{i}_{tag}_mask"]), i
        # nibble legality (SPEC invariants)
        assert set(np.unique(meta)) <= ref.ADMISSIBLE[mode]
        # decompress . compress == prune (test_acceptance.py:67-87)
        pruned, _ = ref.prune_dense(s, mode)
        assert np.array_equal(ref.decompress(nz, meta, s.shape[1], mode), pruned)


def test_fused_identity_kat():
    g = golden("fused.npz")
    eye = np.eye(4)
    for impl in ("numpy", "c"):
        if impl == "numpy":
            nz, meta = ref.sddmm_compress(eye, eye, 1.0, "1:2")
        else:
            nz, meta2d, stats = oracle_c.sddmm_compress(eye, eye, 1.0, "1:2")
            meta = meta2d.ravel()
            assert list(stats) == list(g["identity_stats"])
        assert np.array_equal(nz, g["identity_nonzeros"])
        assert list(meta) == [0x4, 0x4, 0xE, 0x4, 0x4, 0x4, 0x4, 0xE]


def test_fused_cases_bitwise_numpy_and_c():
    g = golden("fused.npz")
    for i in range(int(g["n_cases"])):
        mode = str(g[f"case{i}_mode"])
        q, k, scale = g[f"case{i}_q"], g[f"case{i}_k"], float(g[f"case{i}_scale"])
        nz, meta = ref.sddmm_compress(q, k, scale, mode)
        assert np.array_equal(nz, g[f"case{i}_nonzeros"]), i
        assert np.array_equal(meta, g[f"case{i}_metadata"]), i
        nz_c, meta_c, stats = oracle_c.sddmm_compress(q, k, scale, mode)
        assert np.array_equal(nz_c, g[f"case{i}_nonzeros"]), i
        assert np.array_equal(meta_c.ravel(), g[f"case{i}_metadata"]), i
        assert list(stats) == list(g[f"case{i}_stats"]), i


def test_fused_block_masked_c():
    g = golden("fused.npz")
    nz, meta, stats = oracle_c.sddmm_compress(g["masked_q"], g["masked_k"], 1.0, "1:2", 32, 32,
                                              g["masked_keep"])
    assert np.array_equal(nz, g["masked_nonzeros"])
    assert np.array_equal(meta.ravel(), g["masked_metadata"])
    assert list(stats) == list(g["masked_stats"])


def test_softmax_and_spmm_match_reference():
    g = golden("sparse_ops.npz")
    for i in range(int(g["n_cases"])):
        mode = str(g[f"case{i}_mode"])
        nz, meta, cols = g[f"case{i}_nonzeros"], g[f"case{i}_metadata"], int(g[f"case{i}_dense_cols"])
        want = g[f"case{i}_softmax"]
        sm_c = oracle_c.softmax_nonzeros(nz)
        sm_np = ref.softmax_nonzeros(nz)
        # C restatement calls libm exp like numba: bitwise; numpy's vector exp may differ by 1 ulp
        assert np.array_equal(sm_c, want), i
        assert np.abs(sm_np - want).max() <= 4e-16, i
        colidx = ref.nonzero_columns(meta, nz.shape[0], cols, mode)
        assert np.array_equal(colidx, oracle_c.nonzero_columns(meta, nz.shape[0], cols, mode))
        v = g[f"case{i}_v"]
        assert np.array_equal(oracle_c.spmm_gather(want, colidx, v), g[f"case{i}_spmm"]), i
        assert np.array_equal(ref.spmm_gather(want, colidx, v), g[f"case{i}_spmm"]), i


def test_pipeline_cases():
    g = golden("pipeline.npz")
    for i in range(int(g["n_cases"])):
        q, k, v = g[f"case{i}_q"], g[f"case{i}_k"], g[f"case{i}_v"]
        for mode in ("1:2", "2:4"):
            tag = mode.replace(":", "")
            want = g[f"case{i}_nm{tag}"]
            assert np.array_equal(oracle_c.nm_attention(q, k, v, mode), want), (i, mode)
            assert np.abs(ref.nm_attention(q, k, v, mode) - want).max() <= 1e-14, (i, mode)
            s = ref.gemm_scaled(q, k, 1.0 / np.sqrt(q.shape[1]))
            assert np.array_equal(ref.compress_logical(s, mode)[1], g[f"case{i}_meta{tag}"])


def test_rel_l2_pin_reproduced():
    # test_acceptance.py:227-245 -- seed 20240101, n=256, d=64, 1:2
    g = golden("pipeline.npz")
    q, k, v = g["pin_q"], g["pin_k"], g["pin_v"]
    full = oracle_c.full_attention(q, k, v)
    sparse = oracle_c.nm_attention(q, k, v, "1:2")
    assert np.array_equal(full, g["pin_full"])
    assert np.array_equal(sparse, g["pin_nm12"])
    rel, _, _ = ref.approx_error(full, sparse)
    assert abs(rel - REL_L2_PIN) <= 1e-9


def test_batched_threads_equal_serial():
    rng = np.random.default_rng(5)
    q, k, v = (rng.standard_normal((5, 64, 16)) for _ in range(3))
    for mode in ("1:2", "2:4"):
        got = oracle_c.attention_batched(q, k, v, mode, nthreads=3)
        for h in range(5):
            assert np.array_equal(got[h], oracle_c.nm_attention(q[h], k[h], v[h], mode))
    dense = oracle_c.attention_batched(q, k, v, "1:2", nthreads=2, dense=True)
    assert np.array_equal(dense[1], oracle_c.full_attention(q[1], k[1], v[1]))
