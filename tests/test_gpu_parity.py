"""GPU parity tests: the sm_100a kernels against the CPU oracle (pinned to the reference).

Bars (BASELINE.json north_star):
  * metadata and kept masks BIT-EXACT when the oracle is fed the same score
    tensor the epilogue selected on (the fp32 post-scale dump);
  * nonzeros bit-exact in fp32, equal to the RNE-rounded oracle nonzeros in 16-bit;
  * attention outputs |o - o_ref| <= atol + rtol*|o_ref| with rtol = atol = 1e-5
    (fp32) and 2e-2 (bf16 / fp16), o_ref = reference nm_attention in float64 on
    the same dtype-rounded inputs.
"""

import math

import numpy as np
import pytest
import torch

from conftest import golden
from gpu_helpers import assert_close, logical_meta, oracle_attention, oracle_on_scores, seeded_qkv

import paper_2203_00091_b200 as dfss
from oracle import nmattn_oracle as ref
from oracle import oracle_c

pytestmark = pytest.mark.gpu

M12 = dfss.SparsityMode.ONE_OF_TWO
M24 = dfss.SparsityMode.TWO_OF_FOUR
MODES = {"1:2": M12, "2:4": M24}
TOL = {torch.float32: 1e-5, torch.bfloat16: 2e-2, torch.float16: 2e-2}


def _np(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


# ---------------------------------------------------------------- selection hook


def test_select_group_anchors_on_device():
    g = golden("codec.npz")
    for i in range(int(g["n_groups"])):
        mode = str(g[f"group{i}_mode"])
        vals = g[f"group{i}_values"]
        if not np.array_equal(vals.astype(np.float32).astype(np.float64), vals):
            continue
        sel = dfss.select_group(vals, MODES[mode])
        assert list(sel.kept) == list(g[f"group{i}_kept"]), i
        assert sel.nibble == int(g[f"group{i}_nibble"]), i


@pytest.mark.parametrize("mode", ["1:2", "2:4"])
def test_prune_scores_bitexact_vs_reference(mode):
    g = golden("codec.npz")
    tag = mode.replace(":", "")
    for i in range(int(g["n_scores"])):
        s64 = g[f"scores{i}"]
        s32 = s64.astype(np.float32)
        nz, meta, kept = dfss.prune_scores(torch.from_numpy(s32).cuda(), mode)
        want_nz, want_meta, want_kept = oracle_on_scores(s32.astype(np.float64), mode)
        assert np.array_equal(meta.cpu().numpy(), want_meta), i
        assert np.array_equal(kept.cpu().numpy(), want_kept), i
        assert np.array_equal(_np(nz), want_nz), i
        if np.array_equal(s32.astype(np.float64), s64):  # exactly representable: the reference's own output
            assert np.array_equal(meta.cpu().numpy().ravel(), g[f"scores{i}_{tag}_metadata"]), i
            assert np.array_equal(kept.cpu().numpy(), g[f"scores{i}_{tag}_mask"]), i


def test_prune_scores_16bit_nonzeros_are_rne_of_oracle():
    rng = np.random.default_rng(3)
    s = (rng.standard_normal((64, 256)) * 3).astype(np.float32)
    for dt in (torch.bfloat16, torch.float16):
        nz, meta, _ = dfss.prune_scores(torch.from_numpy(s).cuda(), "2:4", nz_dtype=dt)
        want_nz, want_meta, _ = oracle_on_scores(s.astype(np.float64), "2:4")
        assert np.array_equal(meta.cpu().numpy(), want_meta)
        assert torch.equal(nz.cpu(), torch.from_numpy(want_nz.astype(np.float32)).to(dt))


def test_meta_layout_roundtrip_and_word_formula():
    rng = np.random.default_rng(11)
    for mode, (bh, rows, cols) in [("2:4", (3, 200, 96)), ("1:2", (2, 130, 40)), ("2:4", (1, 256, 512))]:
        m = MODES[mode]
        nibs = np.array(sorted(m.admissible_nibbles), dtype=np.uint8)
        logical = nibs[rng.integers(0, len(nibs), size=(bh, rows, cols // m.group_size))]
        nz = torch.zeros((bh, rows, cols // 2), device="cuda")
        c = dfss.CompressedSparse.from_logical(rows, cols, m, nz, torch.from_numpy(logical).cuda())
        assert np.array_equal(logical_meta(c), logical)
        hw = c.meta_hw.cpu().numpy().view(np.uint32).reshape(bh, -1)
        chunks = -(-(cols // m.group_size) // 8)
        for _ in range(200):  # spot-check the documented word layout (include/dfss.h)
            b = int(rng.integers(bh))
            r = int(rng.integers(rows))
            grp = int(rng.integers(cols // m.group_size))
            rb, rr, cidx, gi = r // 128, r % 128, grp // 8, grp % 8
            lane = 16 * (rr // 16) + 8 * (gi // 4) + rr % 8
            shift = 16 * ((rr // 8) % 2) + 4 * (gi % 4)
            word = hw[b, (rb * chunks + cidx) * 128 + lane]
            assert (int(word) >> shift) & 0xF == logical[b, r, grp]


def test_from_logical_rejects_malformed_nibble():
    nz = torch.zeros((1, 4, 2), device="cuda")
    with pytest.raises(ValueError, match="malformed nibble"):
        dfss.CompressedSparse.from_logical(4, 4, M12, nz, torch.tensor([4, 4, 4, 4, 4, 4, 4, 0x9]))


# ---------------------------------------------------------------- fused SDDMM + prune


SDDMM_SHAPES = [(1, 64, 64, 16), (2, 100, 36, 7), (3, 128, 256, 64), (2, 384, 384, 64), (1, 33, 520, 24)]


@pytest.mark.parametrize("mode", ["1:2", "2:4"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16])
@pytest.mark.parametrize("math_mode", ["auto", "ffma"])
def test_sddmm_same_scores_bitexact(mode, dtype, math_mode):
    m = MODES[mode]
    for bh, n, mk, d in SDDMM_SHAPES:
        if mk % m.group_size:
            continue
        g = torch.Generator().manual_seed(bh * 1000 + n + mk + d)
        q = torch.randn((bh, n, d), generator=g).to(dtype).cuda()
        k = torch.randn((bh, mk, d), generator=g).to(dtype).cuda()
        scale = 1.0 / math.sqrt(d)
        dbg = torch.empty((bh, n, mk), dtype=torch.float32, device="cuda")
        c, stats = dfss.sddmm_prune(q, k, m, scale, scores_out=dbg, math_mode=math_mode)
        assert stats.dense_elems_written == 0
        s = _np(dbg)
        # the dump is the fp32 scaled product (accumulated in fp32)
        exact = np.einsum("bnd,bmd->bnm", _np(q), _np(k)) * scale
        assert_close(s, exact, 1e-5, 1e-5 * max(1.0, float(np.abs(exact).max())), "scores")
        meta = logical_meta(c)
        nz = c.nonzeros
        for b in range(bh):
            want_nz, want_meta, _ = oracle_on_scores(s[b], mode)
            assert np.array_equal(meta[b], want_meta), (bh, n, mk, d, b)
            if c.nonzeros.dtype == torch.float32:
                assert np.array_equal(_np(nz[b]), want_nz)
            else:
                assert torch.equal(nz[b].cpu(), torch.from_numpy(want_nz.astype(np.float32)).to(nz.dtype))


@pytest.mark.parametrize("mode", ["1:2", "2:4"])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("scale", [0.125, 0.1, 1.0, 2.0 ** -7])
def test_sddmm_tcgen05_scales_bitexact(mode, dtype, scale):
    """tcgen05 SDDMM at d = 64 with power-of-two scales (bf16: Q scaled in shared memory, the
    epilogue reads post-scale scores) and other scales (per-score multiply): selection and
    nonzeros bit-exact on the dumped scores, the dump equal to scale * Q K^T within fp32."""
    m = MODES[mode]
    g = torch.Generator().manual_seed(int(scale * 1000) + 7)
    q = torch.randn((2, 256, 64), generator=g).to(dtype).cuda()
    k = torch.randn((2, 384, 64), generator=g).to(dtype).cuda()
    dbg = torch.empty((2, 256, 384), dtype=torch.float32, device="cuda")
    c, _ = dfss.sddmm_prune(q, k, m, scale, scores_out=dbg)
    s = _np(dbg)
    exact = np.einsum("bnd,bmd->bnm", _np(q), _np(k)) * scale
    assert_close(s, exact, 1e-5, 1e-5 * max(1.0, float(np.abs(exact).max())), "scores")
    meta = logical_meta(c)
    for b in range(2):
        want_nz, want_meta, _ = oracle_on_scores(s[b], mode)
        assert np.array_equal(meta[b], want_meta)
        assert torch.equal(c.nonzeros[b].cpu(), torch.from_numpy(want_nz.astype(np.float32)).to(dtype))


def test_sddmm_reference_golden_cases():
    """The reference's own fused instances (fp64) run in fp32: integer-lattice cases are
    exact in fp32 and must match the reference bitwise; the others match the oracle on the
    dumped scores bitwise and the fp64 reference up to near-tie flips (counted)."""
    g = golden("fused.npz")
    flips = total = 0
    for i in range(int(g["n_cases"])):
        mode = str(g[f"case{i}_mode"])
        q64, k64, scale = g[f"case{i}_q"], g[f"case{i}_k"], float(g[f"case{i}_scale"])
        q = torch.from_numpy(q64.astype(np.float32)).cuda()
        k = torch.from_numpy(k64.astype(np.float32)).cuda()
        dbg = torch.empty((q.shape[0], k.shape[0]), dtype=torch.float32, device="cuda")
        c, st = dfss.sddmm_prune(q, k, MODES[mode], scale, scores_out=dbg)
        assert [st.peak_tile_elems, st.nonzeros_written, st.nibbles_written] == list(g[f"case{i}_stats"])
        meta = logical_meta(c).ravel()
        want = oracle_on_scores(_np(dbg), mode)[1].ravel()
        assert np.array_equal(meta, want), i
        integer = np.array_equal(np.round(q64), q64) and np.array_equal(np.round(k64), k64) and scale == 1.0
        if integer:
            assert np.array_equal(meta, g[f"case{i}_metadata"]), i
        flips += int((meta != g[f"case{i}_metadata"]).sum())
        total += meta.size
    assert flips <= max(2, total // 2000), (flips, total)


def test_identity_kat():
    eye = torch.eye(4, device="cuda")
    c, stats = dfss.sddmm_prune(eye, eye, M12, 1.0)
    assert np.array_equal(_np(c.nonzeros), [[1, 0], [1, 0], [0, 1], [0, 1]])
    assert list(c.metadata.cpu().numpy()) == [0x4, 0x4, 0xE, 0x4, 0x4, 0x4, 0x4, 0xE]
    assert stats.nonzeros_written == 8 and stats.nibbles_written == 8


def test_sddmm_block_mask_matches_reference():
    g = golden("fused.npz")
    mask = dfss.BlockMask(g["masked_keep"], tile_rows=32, tile_cols=32)
    q = torch.from_numpy(g["masked_q"].astype(np.float32)).cuda()
    k = torch.from_numpy(g["masked_k"].astype(np.float32)).cuda()
    dbg = torch.empty((64, 64), dtype=torch.float32, device="cuda")
    c, st = dfss.sddmm_prune(q, k, M12, 1.0, mask, tile_rows=32, tile_cols=32, scores_out=dbg)
    assert [st.peak_tile_elems, st.nonzeros_written, st.nibbles_written] == list(g["masked_stats"])
    present = mask.nonzero_keep(64, 64)
    want_nz, want_meta, _ = oracle_on_scores(_np(dbg), "1:2")
    assert np.array_equal(_np(c.nonzeros)[present], want_nz[present])
    assert np.array_equal(logical_meta(c)[present], want_meta[present])
    assert not _np(c.nonzeros)[~present].any()
    assert not logical_meta(c)[~present].any()


@pytest.mark.parametrize("mode", ["2:4", "1:2"])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_masked_sddmm_on_tcgen05_matches_reference(mode, dtype):
    """Block-masked sddmm_prune on the tcgen05 kernel (16-bit, tiled shape): selection bit-exact on
    the dumped scores for present groups, absent groups zero with no metadata (fused.py:73-82)."""
    rng = np.random.default_rng(41)
    n, m = 256, 384
    keep = rng.random((n // 16, m // 16)) < 0.6
    keep[:, 0] = True  # no empty row
    mask = dfss.BlockMask(keep, tile_rows=16, tile_cols=16)
    q = torch.from_numpy(rng.standard_normal((2, n, 64)).astype(np.float32)).to(dtype).cuda()
    k = torch.from_numpy(rng.standard_normal((2, m, 64)).astype(np.float32)).to(dtype).cuda()
    dbg = torch.empty((2, n, m), dtype=torch.float32, device="cuda")
    c, _ = dfss.sddmm_prune(q, k, mode, 0.125, mask, tile_rows=16, tile_cols=16, scores_out=dbg)
    present = mask.nonzero_keep(n, m)
    meta = logical_meta(c)
    for b in range(2):
        want_nz, want_meta, _ = oracle_on_scores(_np(dbg[b]), mode)
        gp = _group_present(present, mode)
        assert np.array_equal(meta[b][gp], want_meta[gp])
        assert not meta[b][~gp].any()
        nzb = c.nonzeros[b].float().cpu().numpy()
        assert np.array_equal(nzb[present], torch.from_numpy(want_nz[present].astype(np.float32)).to(dtype).float().numpy())
        assert not nzb[~present].any()


def _group_present(present_nz: np.ndarray, mode: str) -> np.ndarray:
    """[rows, groups] presence from the [rows, nonzeros] presence (groups never straddle tiles)."""
    per = 2 if mode == "2:4" else 1
    return present_nz[:, ::per]


@pytest.mark.parametrize("mode", ["2:4", "1:2"])
def test_masked_staged_attention_on_tcgen05(mode):
    """nm_attention with a block mask the fused kernel does not tile (16-column tiles) runs the
    staged path -- masked tcgen05 SDDMM, masked softmax, tcgen05 SpMM over the zeroed absent
    entries -- and matches the reference masked pipeline."""
    rng = np.random.default_rng(5)
    n = 512
    keep = rng.random((n // 32, n // 16)) < 0.5
    keep[np.arange(n // 32), np.arange(n // 32) * 2] = True
    mask = dfss.BlockMask(keep, tile_rows=32, tile_cols=16)
    (q, k, v), (q64, k64, v64) = seeded_qkv((1, 2, n, 64), torch.bfloat16, seed=12)
    assert dfss.attention_path(mode, q.dtype, n, 64, block_mask=mask).startswith("staged")
    out = _np(dfss.dfss_attention(q, k, v, mode, block_mask=mask))
    for h in range(2):
        assert_close(out[0, h], _masked_oracle(q64[0, h], k64[0, h], v64[0, h], mask, mode), 2e-2, 2e-2,
                     f"masked staged {mode} head {h}")


# ---------------------------------------------------------------- softmax


def _row(values, mode=M12, dtype=torch.float32):
    values = list(values)
    dense = []
    if mode is M12:
        for v in values:
            dense += [v, min(v - 1.0, -1.0)]
    else:
        for a, b in zip(values[0::2], values[1::2]):
            low = min(a, b) - 1.0
            dense += [a, b, low, low]
    return dfss.compress_logical(torch.tensor([dense], dtype=dtype, device="cuda"), mode)


def test_softmax_kats():
    out = dfss.softmax_rows(_row([0.0, 0.0]))
    assert np.array_equal(_np(out.nonzeros), [[0.5, 0.5]])
    out = dfss.softmax_rows(_row([math.log(3.0), 0.0]))
    assert np.allclose(_np(out.nonzeros), [[0.75, 0.25]], atol=1e-7)
    out = dfss.softmax_rows(_row([1000.0, 1001.0]))
    e = math.e
    assert np.allclose(_np(out.nonzeros), [[1 / (1 + e), e / (1 + e)]], atol=1e-7)
    assert np.isfinite(_np(out.nonzeros)).all()


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_softmax_matches_oracle_rows_sum_to_one(dtype):
    rng = np.random.default_rng(17)
    for cols in (8, 64, 250, 1024, 4096, 12288):
        s = (rng.standard_normal((3, 40, cols)) * 10).astype(np.float32)
        for mode in (M12, M24):
            if cols % mode.group_size:
                continue
            c = dfss.compress_logical(torch.from_numpy(s).to(dtype).cuda(), mode)
            out = dfss.softmax_rows(c)
            got = _np(out.nonzeros)
            want = np.stack([oracle_c.softmax_nonzeros(_np(c.nonzeros[b])) for b in range(3)])
            tol = 1e-6 if dtype == torch.float32 else 8e-3
            assert_close(got, want, tol, tol * 1e-2, f"softmax cols={cols}")
            assert np.abs(got.sum(-1) - 1.0).max() <= (1e-5 if dtype == torch.float32 else 2e-2 * 1)
            # order preservation within each row (ties allowed after rounding)
            assert torch.equal(out.meta_hw, c.meta_hw)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_softmax_16bit_fast_path_edges(dtype):
    """The packed 16-bit softmax (rows of 256 k nonzeros <= 2048, several short rows per warp):
    ragged row counts, every row width it serves, the oracle at 8e-3; a NaN input raises the
    reference's ValueError, an inf input gives NaN without one (numba: exp(inf - inf))."""
    rng = np.random.default_rng(3)
    for rows, nz in ((7, 256), (13, 512), (5, 768), (3, 2048), (130, 256)):
        s = (rng.standard_normal((1, rows, 2 * nz)) * 4).astype(np.float32)
        c = dfss.compress_logical(torch.from_numpy(s).to(dtype).cuda(), M24)
        got = _np(dfss.softmax_rows(c).nonzeros)[0]
        want = oracle_c.softmax_nonzeros(_np(c.nonzeros[0]))
        assert_close(got, want, 8e-3, 8e-5, f"fast softmax rows={rows} nz={nz}")
    c = dfss.compress_logical(torch.randn(1, 4, 512, device="cuda").to(dtype), M24)
    bad = c.nonzeros.clone()
    bad[0, 2, 17] = float("nan")
    with pytest.raises(ValueError, match="NaN"):
        dfss.softmax_rows(dfss.CompressedSparse(c.rows, c.dense_cols, c.mode, bad, c.meta_hw))
    inf = c.nonzeros.clone()
    inf[0, 1, 5] = float("inf")
    out = _np(dfss.softmax_rows(dfss.CompressedSparse(c.rows, c.dense_cols, c.mode, inf, c.meta_hw)).nonzeros)
    assert np.isnan(out[0, 1]).any() and np.isfinite(out[0, 0]).all()


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("tiles", [(32, 16), (16, 64), (64, 48), (32, 8)])
def test_softmax_16bit_block_mask(dtype, tiles):
    """softmax_rows with a BlockMask on 16-bit rows: tile widths that are multiples of 16 run the
    packed fast path (absent vectors -inf before the max), 8 the generic kernel; both equal the
    reference softmax over the present entries (absent -> 0) at 8e-3; NaN in an absent entry is
    ignored, in a present one raises."""
    rng = np.random.default_rng(tiles[0] * 100 + tiles[1])
    tr, tc_ = tiles
    for rows, nz in ((96, 256), (64, 1024), (32, 2048)):
        keep = rng.random((-(-rows // tr), -(-2 * nz // tc_))) < 0.5
        keep[np.arange(keep.shape[0]), rng.integers(0, keep.shape[1], keep.shape[0])] = True
        mask = dfss.BlockMask(keep, tile_rows=tr, tile_cols=tc_)
        s = (rng.standard_normal((2, rows, 2 * nz)) * 4).astype(np.float32)
        c = dfss.compress_logical(torch.from_numpy(s).to(dtype).cuda(), M24)
        present = mask.nonzero_keep(rows, 2 * nz)
        nzv = c.nonzeros.clone()
        nzv[:, torch.from_numpy(~present).cuda()] = float("nan")  # absent entries are never read
        cm = dfss.CompressedSparse(rows, 2 * nz, c.mode, nzv, c.meta_hw, block_mask=mask)
        got = _np(dfss.softmax_rows(cm).nonzeros)
        for b in range(2):
            want = oracle_c.softmax_nonzeros(_np(c.nonzeros[b]), present)
            assert_close(got[b], want, 8e-3, 8e-5, f"masked softmax tiles={tiles} rows={rows} nz={nz}")
            assert not got[b][~present].any()
        bad = nzv.clone()
        r, j = np.argwhere(present)[len(np.argwhere(present)) // 2]
        bad[1, r, j] = float("nan")
        with pytest.raises(ValueError, match="NaN"):
            dfss.softmax_rows(dfss.CompressedSparse(rows, 2 * nz, c.mode, bad, c.meta_hw, block_mask=mask))


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_staged_12_tcgen05_attention_matches_reference(dtype):
    """1:2 through the staged reference-shaped API on the tcgen05 kernels (16-bit, tiled shape):
    sddmm_prune -> softmax_rows -> spmm equals the reference nm_attention at 2e-2."""
    (q, k, v), (q64, k64, v64) = seeded_qkv((1, 3, 1024, 64), dtype, seed=8)
    c, _ = dfss.sddmm_prune(q, k, "1:2", 0.125)
    out = _np(dfss.spmm(dfss.softmax_rows(c), v).data)
    assert_close(out, oracle_attention(q64, k64, v64, "1:2"), 2e-2, 2e-2, "staged 1:2 tcgen05")


def test_softmax_rejects_nan_and_empty_rows():
    c = _row([0.0, 1.0])
    bad = dfss.CompressedSparse(c.rows, c.dense_cols, c.mode, torch.tensor([[float("nan"), 1.0]], device="cuda"),
                                c.meta_hw)
    with pytest.raises(ValueError, match="NaN"):
        dfss.softmax_rows(bad)
    q = torch.randn(64, 4, device="cuda")
    mask = dfss.BlockMask(np.array([[False], [True]]), tile_rows=32, tile_cols=64)
    cm, _ = dfss.sddmm_prune(q, q, M12, 1.0, mask)
    with pytest.raises(ValueError, match="empty row 0"):
        dfss.softmax_rows(cm)


# ---------------------------------------------------------------- SpMM


def test_spmm_single_nonzero_kat():
    nonzeros = torch.zeros((3, 2), device="cuda")
    nonzeros[1, 1] = 2.5
    meta = torch.tensor([0x4, 0x4, 0x4, 0xE, 0x4, 0x4], dtype=torch.uint8)
    c = dfss.CompressedSparse.from_logical(3, 4, M12, nonzeros, meta)
    v = torch.arange(8.0, device="cuda").reshape(4, 2)
    out = dfss.spmm(c, v).data
    assert torch.equal(out[1], 2.5 * v[3])
    assert not out[[0, 2]].any()


@pytest.mark.parametrize("mode", ["1:2", "2:4"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16])
def test_spmm_matches_decompress_oracle(mode, dtype):
    rng = np.random.default_rng(23)
    m = MODES[mode]
    for bh, rows, cols, d in [(1, 4, 8, 3), (2, 64, 64, 16), (2, 128, 512, 64), (3, 256, 384, 64), (1, 96, 200, 40)]:
        if cols % m.group_size:
            continue
        a = dfss.compress_logical(torch.from_numpy(rng.standard_normal((bh, rows, cols)).astype(np.float32))
                                  .to(dtype).cuda(), m)
        p = dfss.softmax_rows(a)
        v = torch.from_numpy(rng.standard_normal((bh, cols, d)).astype(np.float32)).to(dtype).cuda()
        out = _np(dfss.spmm(p, v).data)
        nzp = _np(p.nonzeros)
        meta = logical_meta(p)
        for b in range(bh):
            colidx = ref.nonzero_columns(meta[b].ravel(), rows, cols, mode)
            want = oracle_c.spmm_gather(nzp[b], colidx, _np(v[b]))
            tol = 1e-5 if dtype == torch.float32 else 1e-2
            assert_close(out[b], want, tol, tol, f"spmm {bh, rows, cols, d}")


@pytest.mark.parametrize("mode", ["1:2", "2:4"])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("tiles", [(32, 16), (16, 8), (64, 64), (128, 6)])
def test_spmm_block_mask_tcgen05(mode, dtype, tiles):
    """spmm with a BlockMask on the tcgen05 kernel (16-bit, d = 64): absent nonzeros -- NaN here --
    are zeroed in shared memory before the MMAs (whole 16-byte units for tile widths that are
    multiples of 16, element-wise otherwise), so the output equals the reference gather over the
    present entries (sparse_ops.py:57-64)."""
    rng = np.random.default_rng(tiles[0] + tiles[1])
    tr, tc_ = tiles
    bh, rows, cols = 2, 256, 512
    if tc_ % 2 or (mode == "2:4" and tc_ % 4):
        pytest.skip("tile width must hold whole groups")
    m = MODES[mode]
    keep = rng.random((-(-rows // tr), -(-cols // tc_))) < 0.5
    mask = dfss.BlockMask(keep, tile_rows=tr, tile_cols=tc_)
    a = dfss.compress_logical(torch.from_numpy(rng.standard_normal((bh, rows, cols)).astype(np.float32) / 4)
                              .to(dtype).cuda(), m)
    present = mask.nonzero_keep(rows, cols)
    nz = a.nonzeros.clone()
    nz[:, torch.from_numpy(~present).cuda()] = float("nan")
    p = dfss.CompressedSparse(rows, cols, a.mode, nz, a.meta_hw, block_mask=mask)
    v = torch.from_numpy(rng.standard_normal((bh, cols, 64)).astype(np.float32)).to(dtype).cuda()
    out = _np(dfss.spmm(p, v).data)
    meta = logical_meta(a)
    for b in range(bh):
        colidx = ref.nonzero_columns(meta[b].ravel(), rows, cols, mode)
        want = oracle_c.spmm_gather(_np(a.nonzeros[b]), colidx, _np(v[b]), present)
        assert_close(out[b], want, 1e-2, 1e-2, f"masked spmm {mode} tiles={tiles}")


def test_spmm_linear_in_v():
    a = dfss.compress_logical(torch.randn(8, 8, device="cuda"), M12)
    v = torch.randn(8, 5, device="cuda")
    assert torch.allclose(dfss.spmm(a, 3.0 * v).data, 3.0 * dfss.spmm(a, v).data, rtol=1e-6, atol=1e-6)


# ---------------------------------------------------------------- end to end


def test_c1_fp32_attention_within_1e5():
    """BASELINE config 1: DFSS 1:2 fp32, [1,12,384,64], vs the reference at rtol=atol=1e-5."""
    (q, k, v), (q64, k64, v64) = seeded_qkv((1, 12, 384, 64), torch.float32, seed=0)
    out = dfss.dfss_attention(q, k, v, "1:2")
    want = oracle_attention(q64, k64, v64, "1:2")
    assert_close(_np(out), want, 1e-5, 1e-5, "c1 fp32 1:2")


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("mode", ["2:4", "1:2"])
@pytest.mark.parametrize("n", [512, 384, 128, 1024])
def test_16bit_attention_within_2e2(dtype, mode, n):
    (q, k, v), (q64, k64, v64) = seeded_qkv((2, 3, n, 64), dtype, seed=1)
    out = dfss.dfss_attention(q, k, v, mode)
    want = oracle_attention(q64, k64, v64, mode)
    assert_close(_np(out), want, 2e-2, 2e-2, f"{dtype} {mode} n={n}")


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_flash_kernel_matches_staged_pipeline(dtype):
    """dfss_attention (one fused kernel) vs the staged sddmm -> softmax -> spmm kernels on the
    same inputs: identical selection, so the outputs agree to 16-bit rounding."""
    (q, k, v), _ = seeded_qkv((3, 2, 768, 64), dtype, seed=9)
    flash = _np(dfss.dfss_attention(q, k, v, "2:4"))
    c, _ = dfss.attention_sddmm(q, k, "2:4")
    staged = _np(dfss.spmm(dfss.softmax_rows(c), v).data)
    assert_close(flash, staged, 2e-2, 2e-2, "flash vs staged")
    assert np.abs(flash - staged).max() <= 1.5e-2


def _flash_vs_oracle(q, k, v, what, tol=2e-2):
    """dfss_attention on 16-bit [b, h, n, 64] CUDA tensors vs the reference nm_attention (float64)."""
    out = _np(dfss.dfss_attention(q, k, v, "2:4"))
    want = oracle_attention(*(x.double().cpu().numpy() for x in (q, k, v)), "2:4")
    assert_close(out, want, tol, tol, what)
    return out, want


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_flash_shift_update_path(dtype):
    """Scores that grow along the key axis (later tiles exceed the first tile's maximum by far
    more than 2^8 in probability mass): the lazy-shift slow path must rescale O and the sums."""
    g = torch.Generator().manual_seed(21)
    n = 1024
    q = torch.randn((1, 2, n, 64), generator=g)
    k = torch.randn((1, 2, n, 64), generator=g) * torch.linspace(0.2, 3.0, n).view(1, 1, n, 1)
    v = torch.randn((1, 2, n, 64), generator=g)
    q, k, v = (x.to(dtype).cuda() for x in (q, k, v))
    _flash_vs_oracle(q, k, v, "growing scores")
    # and the reverse: the first tile holds the maximum
    _flash_vs_oracle(q, k.flip(-2).contiguous(), v, "decaying scores")


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_flash_large_logits(dtype):
    """Logits of magnitude ~60: exp spans far beyond fp32 without the shift."""
    (q, k, v), _ = seeded_qkv((1, 3, 512, 64), dtype, seed=5)
    _flash_vs_oracle(q * 8, k, v, "large logits")


@pytest.mark.parametrize("scales", [(0.02, 1.0, 20.0), (1.0, 5.0, 1.0)])
@pytest.mark.parametrize("mode", ["2:4", "1:2"])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_flash_start_shift_carried_across_items(mode, dtype, scales):
    """Unmasked items start their lazy shift from the shift the row ended the CTA's previous item
    with.  Heads whose logit scales jump by 1000x from one item to the next (so each CTA's next
    item starts far too high or far too low) must still match the reference: the first step's
    sums leave [2^-16, 2^8] and it recomputes with the exact row maximum."""
    b, h, n = 2, 150, 512  # 600 items: ~4 per persistent CTA, neighbours on a CTA are 148 apart
    (q, k, v), _ = seeded_qkv((b, h, n, 64), dtype, seed=31)
    # (1, 5, 1): a start shift ~15 too high in log2 units -- fp16 P would sink into the denormal
    # range without the fp16 sum floor (2^-6)
    scale = torch.tensor([[scales[(i * 7 + j) % 3] for j in range(h)] for i in range(b)])
    q = (q.float() * scale.view(b, h, 1, 1).cuda()).to(dtype)
    out = _np(dfss.dfss_attention(q, k, v, mode))
    heads = [(0, 0), (0, 1), (0, 2), (1, 74), (1, 148), (1, 149)]
    for bi, hi in heads:
        want = oracle_attention(*(x[bi, hi].double().cpu().numpy() for x in (q, k, v)), mode)
        assert_close(out[bi, hi], want, 2e-2, 2e-2, f"carried shift {mode} head ({bi},{hi})")


def test_flash_tie_lattice_and_zero_queries():
    """Integer-lattice Q/K (exact bf16, many tied scores) and all-zero queries (every score is
    a signed zero: the reference keeps the lower index of every tie, so O = mean of V rows
    4g, 4g+1)."""
    g = torch.Generator().manual_seed(3)
    n = 512
    q = torch.randint(-1, 2, (1, 2, n, 64), generator=g).to(torch.bfloat16).cuda()
    k = torch.randint(-1, 2, (1, 2, n, 64), generator=g).to(torch.bfloat16).cuda()
    v = torch.randn((1, 2, n, 64), generator=g).to(torch.bfloat16).cuda()
    _flash_vs_oracle(q, k, v, "tie lattice")
    z = torch.zeros_like(q)
    out, want = _flash_vs_oracle(z, k, v, "zero queries")
    vv = v.double().cpu().numpy()[0]
    kept = vv.reshape(2, n // 4, 4, 64)[:, :, :2].reshape(2, n // 2, 64).mean(1)
    assert np.abs(want[0] - kept[:, None, :]).max() < 1e-12
    assert np.abs(out[0] - kept[:, None, :]).max() < 2e-2
    # -0 queries against keys whose sign alternates per key: every dot product is a sum of
    # -0 (or +0) terms only, so in IEEE arithmetic the scores alternate -0 / +0.  The fused
    # kernel relies on tcgen05 writing zero sums as +0 (tools/negzero_probe.cu) to skip
    # canonicalising the pair differences; the reference treats -0 == +0 (lower index wins).
    sign = torch.where(torch.arange(n) % 2 == 0, 1.0, -1.0).view(1, 1, n, 1)
    kpos = (torch.rand((1, 2, n, 64), generator=g) + 0.5) * sign
    out, want = _flash_vs_oracle(-torch.zeros_like(q), kpos.to(torch.bfloat16).cuda(), v, "signed-zero scores")
    assert np.abs(out[0] - kept[:, None, :]).max() < 2e-2


@pytest.mark.parametrize("n", [128, 256, 4096])
def test_flash_sequence_lengths(n):
    (q, k, v), _ = seeded_qkv((1, 2, n, 64), torch.bfloat16, seed=n)
    _flash_vs_oracle(q, k, v, f"n={n}")


@pytest.mark.parametrize("mode", ["2:4", "1:2"])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_fused_softmax_spmm_matches_staged_and_oracle(dtype, mode):
    """spmm_softmax(sddmm_prune(with_row_max)) == spmm(softmax_rows(.)) == reference nm_attention
    (1:2 runs the tcgen05 kernels too: one survivor per pair as the 2:4 pattern 8 + a + 4b)."""
    (q, k, v), (q64, k64, v64) = seeded_qkv((2, 2, 640, 64), dtype, seed=4)
    dbg = torch.empty((2, 2, 640, 640), dtype=torch.float32, device="cuda")
    c, _ = dfss.sddmm_prune(q, k, mode, 0.125, with_row_max=True, scores_out=dbg)
    meta = logical_meta(c)
    for b in range(2):
        for h in range(2):
            _, want_meta, _ = oracle_on_scores(_np(dbg[b, h]), mode)
            assert np.array_equal(meta[b, h], want_meta), (mode, b, h)
    # the recorded row maximum is the exact fp32 max of the row's scores (always a kept value)
    assert torch.equal(c.row_max.amax(-1), dbg.amax(-1))
    fused = _np(dfss.spmm_softmax(c, v).data)
    staged = _np(dfss.spmm(dfss.softmax_rows(c), v).data)
    assert_close(fused, staged, 2e-2, 2e-2, "fused vs staged")
    want = oracle_attention(q64, k64, v64, mode)
    assert_close(fused, want, 2e-2, 2e-2, "fused vs oracle")


def test_golden_pipeline_cases_fp32():
    g = golden("pipeline.npz")
    for i in range(int(g["n_cases"])):
        q64, k64, v64 = g[f"case{i}_q"], g[f"case{i}_k"], g[f"case{i}_v"]
        to = lambda x: torch.from_numpy(x.astype(np.float32)).cuda()
        for mode in ("1:2", "2:4"):
            inputs = dfss.AttentionInputs(dfss.DenseMatrix(to(q64)), dfss.DenseMatrix(to(k64)), dfss.DenseMatrix(to(v64)))
            out = _np(dfss.nm_attention(inputs, MODES[mode]).data)
            want = oracle_c.nm_attention(*(x.astype(np.float32).astype(np.float64) for x in (q64, k64, v64)), mode)
            assert_close(out, want, 1e-5, 1e-5, f"golden case {i} {mode}")


def test_rel_l2_pin_on_device():
    g = golden("pipeline.npz")
    to = lambda x: torch.from_numpy(x.astype(np.float32)).cuda()
    inputs = dfss.AttentionInputs(*(dfss.DenseMatrix(to(g[f"pin_{c}"])) for c in "qkv"))
    err = dfss.approx_error(torch.from_numpy(g["pin_full"]).cuda(), dfss.nm_attention(inputs, M12))
    assert abs(err.rel_l2 - 0.39969464809566535) <= 1e-5


def test_identical_keys_and_single_token():
    n, d = 8, 4
    k_row = torch.randn(d)
    q = torch.randn(n, d, device="cuda")
    k = k_row.repeat(n, 1).cuda()
    v = torch.randn(n, d, device="cuda")
    out = dfss.nm_attention(dfss.AttentionInputs(q, k, v), M12).data
    assert torch.allclose(out, v[0::2].mean(0).expand(n, d), rtol=1e-5, atol=1e-6)
    q1, k1, v1, vp = (torch.randn(1, 8, device="cuda") for _ in range(4))
    out = dfss.nm_attention(dfss.AttentionInputs(torch.cat([q1, q1]), torch.cat([k1, k1]), torch.cat([v1, vp])), M12)
    assert torch.equal(out.data[0], v1[0])


def test_block_masked_pipeline_matches_staged_oracle():
    rng = np.random.default_rng(5)
    n, d = 64, 8
    q64, k64, v64 = (rng.standard_normal((n, d)).astype(np.float32).astype(np.float64) for _ in range(3))
    keep = np.array([[True, False], [True, True]])
    mask = dfss.BlockMask(keep, tile_rows=32, tile_cols=32)
    to = lambda x: torch.from_numpy(x.astype(np.float32)).cuda()
    out = _np(dfss.nm_attention(dfss.AttentionInputs(to(q64), to(k64), to(v64)), M12, mask, tile_rows=32,
                                tile_cols=32).data)
    scores = ref.gemm_scaled(q64, k64, 1.0 / math.sqrt(d))
    nz, meta = ref.compress_logical(scores, "1:2")
    present = mask.nonzero_keep(n, n)
    p = oracle_c.softmax_nonzeros(nz, present)
    cols = ref.nonzero_columns(meta, n, n, "1:2")
    want = oracle_c.spmm_gather(p, cols, v64, present)
    assert_close(out, want, 1e-5, 1e-5, "masked pipeline")


def _masked_oracle(q64, k64, v64, mask, mode):
    """Reference nm_attention with a block mask (fused.py:73-82, sparse_ops.py:18-68) on one head."""
    n, d = q64.shape
    scores = ref.gemm_scaled(q64, k64, 1.0 / math.sqrt(d))
    nz, meta = ref.compress_logical(scores, mode)
    present = mask.nonzero_keep(n, n)
    p = oracle_c.softmax_nonzeros(nz, present)
    cols = ref.nonzero_columns(meta, n, n, mode)
    return oracle_c.spmm_gather(p, cols, v64, present)


@pytest.mark.parametrize("n,tiles,mode,dtype", [
    (512, (32, 64), "2:4", torch.bfloat16),   # two-set fused kernel, reference default tiling
    (512, (64, 128), "1:2", torch.float16),   # two-set, coarser tiles, 1:2
    (384, (32, 32), "2:4", torch.float16),    # one-set fused kernel (n % 256 != 0)
    (256, (16, 64), "2:4", torch.bfloat16),   # tile rows not 32-aligned: staged kernels
])
def test_block_masked_attention_matches_reference(n, tiles, mode, dtype):
    """BlockMask on the fast path: masked tiles structurally absent, softmax over the present
    kept entries, per head; includes row blocks whose first key tiles are masked."""
    rng = np.random.default_rng(n)
    tr, tc_ = tiles
    keep = rng.random((-(-n // tr), -(-n // tc_))) < 0.55
    keep[:, 0] = False          # first key tile masked everywhere: the shift starts at -inf
    keep[np.arange(keep.shape[0]), rng.integers(1, keep.shape[1], keep.shape[0])] = True  # no empty row
    mask = dfss.BlockMask(keep, tile_rows=tr, tile_cols=tc_)
    (q, k, v), (q64, k64, v64) = seeded_qkv((1, 2, n, 64), dtype, seed=7)
    out = _np(dfss.dfss_attention(q, k, v, mode, block_mask=mask))
    for h in range(2):
        want = _masked_oracle(q64[0, h], k64[0, h], v64[0, h], mask, mode)
        assert_close(out[0, h], want, 2e-2, 2e-2, f"masked {mode} n={n} tiles={tiles} head {h}")
    # nm_attention with the reference signature routes to the same path
    got = _np(dfss.nm_attention(dfss.AttentionInputs(q[0, 0], k[0, 0], v[0, 0]), mode, mask, tile_rows=tr,
                                tile_cols=tc_).data)
    assert_close(got, out[0, 0], 1e-6, 1e-6, "nm_attention(block_mask) == dfss_attention(block_mask)")


def _block_causal_keep(n, tr, tc_, blk=128):
    """Keep-mask on (tr, tc_) tiles that is block-causal at blk x blk granularity."""
    rows = np.arange(-(-n // tr)) * tr // blk
    cols = np.arange(-(-n // tc_)) * tc_ // blk
    return cols[None, :] <= rows[:, None]


@pytest.mark.parametrize("mode,dtype", [("2:4", torch.bfloat16), ("1:2", torch.float16)])
def test_block_mask_whole_steps_skipped(mode, dtype):
    """Whole 128 x 128 steps masked (block-causal + random dead blocks): the two-set kernel skips
    them entirely, including steps dead for one 128-row half of a 256-row item only; several
    items per CTA so the barrier phases must survive variable step counts."""
    n, tr, tc_ = 1024, 32, 64
    rng = np.random.default_rng(11)
    keep = _block_causal_keep(n, tr, tc_)
    blocks = rng.random((n // 128, n // 128)) < 0.3          # extra dead 128 x 128 blocks below the diagonal
    np.fill_diagonal(blocks, False)
    keep &= ~np.kron(blocks, np.ones((128 // tr, 128 // tc_), dtype=bool))
    mask = dfss.BlockMask(keep, tile_rows=tr, tile_cols=tc_)
    (q, k, v), (q64, k64, v64) = seeded_qkv((4, 40, n, 64), dtype, seed=5)   # 640 items > 148 CTAs
    out = _np(dfss.dfss_attention(q, k, v, mode, block_mask=mask))
    for b, h in [(0, 0), (1, 17), (3, 39)]:
        want = _masked_oracle(q64[b, h], k64[b, h], v64[b, h], mask, mode)
        assert_close(out[b, h], want, 2e-2, 2e-2, f"block-causal {mode} ({b},{h})")


def test_block_mask_skipping_saves_time():
    """Block-causal masks (~56% of the 128 x 128 steps live at n = 4096) cut the fused kernel time."""
    n = 4096
    (q, k, v), _ = seeded_qkv((1, 64, n, 64), torch.bfloat16, seed=3)
    mask = dfss.BlockMask(_block_causal_keep(n, 32, 64), 32, 64)
    out = torch.empty_like(q)

    def timed(bm):
        for _ in range(3):
            dfss.dfss_attention(q, k, v, "2:4", block_mask=bm, out=out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            dfss.dfss_attention(q, k, v, "2:4", block_mask=bm, out=out)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 10

    dense, causal = timed(None), timed(mask)
    assert causal < 0.75 * dense, (causal, dense)


def test_block_mask_empty_row_and_tiling_errors():
    (q, k, v), _ = seeded_qkv((1, 1, 256, 64), torch.bfloat16, seed=2)
    keep = np.ones((8, 4), dtype=bool)
    keep[3] = False
    with pytest.raises(ValueError, match="empty row 96"):
        dfss.dfss_attention(q, k, v, "2:4", block_mask=dfss.BlockMask(keep, 32, 64))
    with pytest.raises(ValueError, match="does not match"):
        dfss.dfss_attention(q, k, v, "2:4", block_mask=dfss.BlockMask(np.ones((4, 4), dtype=bool), 32, 64))
    with pytest.raises(ValueError, match="fused tiling"):
        dfss.nm_attention(dfss.AttentionInputs(q[0, 0], k[0, 0], v[0, 0]), "2:4",
                          dfss.BlockMask(np.ones((8, 4), dtype=bool), 32, 64), tile_rows=32, tile_cols=32)


@pytest.mark.parametrize("name,mode", [("12", "1:2"), ("24", "2:4")])
def test_container_export_import_bytewise_vs_reference(name, mode, tmp_path):
    """GPU CompressedSparse -> NMCS bytes identical to the reference's to_bytes on the same
    scores (tests/golden/make_container_golden.py); import of the reference file round-trips."""
    g = golden("container.npz")
    scores = torch.from_numpy(g[f"scores_{name}"].astype(np.float32)).cuda()
    want = g[f"nmcs_{name}"].tobytes()
    c = dfss.compress_logical(scores, mode)
    assert dfss.to_bytes(c) == want
    path = tmp_path / "m.nmcs"
    assert dfss.write_container(c, path) == len(want)
    back = dfss.read_container(path)
    assert torch.equal(back.metadata, c.metadata)
    assert torch.equal(back.nonzeros, c.nonzeros)
    assert dfss.to_bytes(back) == want
    # batched export: one slice per container
    cb = dfss.compress_logical(torch.stack([scores, scores]), mode)
    assert dfss.to_bytes(cb, index=1) == want
    with pytest.raises(ValueError, match="index"):
        dfss.to_bytes(cb)


def _tf32(x: np.ndarray) -> np.ndarray:
    """The operand the tf32 tensor core multiplies: fp32 with the low 13 mantissa bits dropped."""
    return (x.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32).astype(np.float64)


@pytest.mark.parametrize("n", [128, 256, 384, 512, 640, 1024])
def test_tf32_12_fused_attention(n):
    """configs[4] "1:2 tf32": fp32 inputs, tf32 tensor cores, fused 1:2 kernel.  Checked like the
    16-bit paths: the reference nm_attention in float64 on the operands the hardware multiplies
    (tf32-truncated Q, K, V), at the 16-bit bar 2e-2; and within 5e-2 of the exact-FP32 pipeline
    (pairs whose scores differ by less than the tf32 rounding may keep the other element)."""
    (q, k, v), (q64, k64, v64) = seeded_qkv((1, 3, n, 64), torch.float32, seed=n + 1)
    out = _np(dfss.dfss_attention(q, k, v, "1:2", math_mode="tf32"))
    want = oracle_attention(_tf32(q64), _tf32(k64), _tf32(v64), "1:2")
    assert_close(out, want, 2e-2, 2e-2, f"tf32 1:2 n={n}")
    exact = _np(dfss.dfss_attention(q, k, v, "1:2", math_mode="ffma"))
    assert np.abs(out - exact).max() < 5e-2


def test_tf32_12_masked_and_shift_path():
    g = torch.Generator().manual_seed(31)
    n = 512
    q = torch.randn((1, 2, n, 64), generator=g)
    k = torch.randn((1, 2, n, 64), generator=g) * torch.linspace(0.2, 3.0, n).view(1, 1, n, 1)
    v = torch.randn((1, 2, n, 64), generator=g)
    q, k, v = (x.cuda() for x in (q, k, v))
    out = _np(dfss.dfss_attention(q, k, v, "1:2", math_mode="tf32"))
    want = oracle_attention(*(_tf32(x.cpu().numpy()) for x in (q, k, v)), "1:2")
    assert_close(out, want, 2e-2, 2e-2, "tf32 growing scores")
    rng = np.random.default_rng(4)
    keep = rng.random((n // 32, n // 64)) < 0.6
    keep[:, 0] = False
    keep[np.arange(keep.shape[0]), rng.integers(1, keep.shape[1], keep.shape[0])] = True
    mask = dfss.BlockMask(keep, 32, 64)
    out = _np(dfss.dfss_attention(q, k, v, "1:2", math_mode="tf32", block_mask=mask))
    qq, kk, vv = (_tf32(x.cpu().numpy()) for x in (q, k, v))
    for h in range(2):
        assert_close(out[0, h], _masked_oracle(qq[0, h], kk[0, h], vv[0, h], mask, "1:2"), 2e-2, 2e-2, "tf32 masked")
    with pytest.raises(RuntimeError, match="tf32 attention needs"):
        dfss.dfss_attention(q, k, v, "2:4", math_mode="tf32")


def test_module_and_value_envelope():
    mod = dfss.DFSSAttention("2:4")
    q, k, v = (torch.randn(2, 4, 256, 64, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    out = mod(q, k, v).float()
    lo = v.float().amin(dim=-2, keepdim=True) - 2e-2
    hi = v.float().amax(dim=-2, keepdim=True) + 2e-2
    assert bool(((out >= lo) & (out <= hi)).all())


def test_heatmap_kept_entries_dominate_dense():
    q, k, v = (torch.randn(64, 16, device="cuda") for _ in range(3))
    for mode in (M12, M24):
        pair = dfss.attention_heatmap(dfss.AttentionInputs(q, k, v), mode)
        kept = pair.sparse.data != 0
        assert bool((pair.sparse.data[kept] >= pair.dense.data[kept] - 1e-6).all())


def test_tf32_12_block_mask_whole_steps_skipped():
    """tf32 kernel with whole 128 x 128 steps masked (block-causal + dead blocks), steps dead
    for one half only, several items per CTA."""
    n, tr, tc_ = 1024, 32, 64
    rng = np.random.default_rng(12)
    keep = _block_causal_keep(n, tr, tc_)
    blocks = rng.random((n // 128, n // 128)) < 0.3
    np.fill_diagonal(blocks, False)
    keep &= ~np.kron(blocks, np.ones((128 // tr, 128 // tc_), dtype=bool))
    keep[:, :2] &= rng.random((keep.shape[0], 2)) < 0.5   # partially masked live steps too
    keep[np.arange(keep.shape[0]), np.arange(keep.shape[0]) * tr // tc_] = True  # diagonal tile: no empty row
    mask = dfss.BlockMask(keep, tile_rows=tr, tile_cols=tc_)
    g = torch.Generator().manual_seed(13)
    q, k, v = (torch.randn((2, 80, n, 64), generator=g).cuda() for _ in range(3))   # 320 items > 148 CTAs
    out = _np(dfss.dfss_attention(q, k, v, "1:2", math_mode="tf32", block_mask=mask))
    for b, h in [(0, 0), (1, 41), (1, 79)]:
        qq, kk, vv = (_tf32(x[b, h].cpu().numpy()) for x in (q, k, v))
        assert_close(out[b, h], _masked_oracle(qq, kk, vv, mask, "1:2"), 2e-2, 2e-2, f"tf32 block-causal ({b},{h})")


def test_tf32_12_odd_row_block_masked_and_many_items():
    """n % 256 == 128: the last 256-row item has an empty second half (treated like a fully
    masked one).  Many items per CTA, with and without a block mask, guard the output rows."""
    n = 384
    g = torch.Generator().manual_seed(17)
    q, k, v = (torch.randn((4, 100, n, 64), generator=g).cuda() for _ in range(3))   # 200 items
    out = torch.full_like(q, float("nan"))
    dfss.dfss_attention(q, k, v, "1:2", math_mode="tf32", out=out)
    assert torch.isfinite(out).all()
    for b, h in [(0, 0), (3, 99)]:
        qq, kk, vv = (_tf32(x[b, h].cpu().double().numpy()) for x in (q, k, v))
        assert_close(_np(out[b, h]), oracle_attention(qq, kk, vv, "1:2"), 2e-2, 2e-2, f"tf32 n=384 ({b},{h})")
    keep = _block_causal_keep(n, 32, 64)
    mask = dfss.BlockMask(keep, 32, 64)
    out = _np(dfss.dfss_attention(q, k, v, "1:2", math_mode="tf32", block_mask=mask))
    for b, h in [(1, 5), (2, 77)]:
        qq, kk, vv = (_tf32(x[b, h].cpu().double().numpy()) for x in (q, k, v))
        assert_close(out[b, h], _masked_oracle(qq, kk, vv, mask, "1:2"), 2e-2, 2e-2, f"tf32 masked n=384 ({b},{h})")


@pytest.mark.parametrize("kind", ["2:4-bf16", "1:2-f16", "1:2-tf32"])
def test_block_mask_one_half_runs_ahead(kind):
    """Rows 0-127 of every 256-row item keep only the last 128 keys, rows 128-255 keep all: one
    softmax set runs every step while the other waits for the item's last step.  A shared S-slot
    barrier would complete two phases past the waiting set (parity aliasing); per-half S
    barriers keep the waits exact."""
    mode, dt = kind.split("-")
    n, tr, tc_ = 1024, 32, 64
    rows = np.arange(n // tr) * tr
    cols = np.arange(n // tc_) * tc_
    keep = np.where(((rows % 256) < 128)[:, None], (cols >= n - 128)[None, :], True)
    mask = dfss.BlockMask(keep, tr, tc_)
    g = torch.Generator().manual_seed(23)
    dtype = {"bf16": torch.bfloat16, "f16": torch.float16, "tf32": torch.float32}[dt]
    q, k, v = (torch.randn((2, 96, n, 64), generator=g).to(dtype).cuda() for _ in range(3))  # 768 items
    kw = {"math_mode": "tf32"} if dt == "tf32" else {}
    out = _np(dfss.dfss_attention(q, k, v, mode, block_mask=mask, **kw))
    for b, h in [(0, 3), (1, 95)]:
        ops = [x[b, h].cpu().double().numpy() for x in (q, k, v)]
        if dt == "tf32":
            ops = [_tf32(x) for x in ops]
        assert_close(out[b, h], _masked_oracle(*ops, mask, mode), 2e-2, 2e-2, f"{kind} skewed mask ({b},{h})")


@pytest.mark.parametrize("pinned", [True, False])
def test_host_api_matches_device_api(pinned):
    """dfss_attention_host (host tensors in / out, pipelined copies) equals dfss_attention on the
    same inputs, for uneven pieces, a block mask and the tf32 path."""
    g = torch.Generator().manual_seed(29)
    q, k, v = (torch.randn((3, 7, 512, 64), generator=g).to(torch.bfloat16) for _ in range(3))
    if pinned:
        q, k, v = (x.pin_memory() for x in (q, k, v))
    want = dfss.dfss_attention(q.cuda(), k.cuda(), v.cuda(), "2:4").cpu()
    got = dfss.dfss_attention_host(q, k, v, "2:4", chunks=5)
    torch.cuda.synchronize()
    assert not got.is_cuda and torch.equal(got, want)
    mask = dfss.BlockMask(_block_causal_keep(512, 32, 64), 32, 64)
    want = dfss.dfss_attention(q.cuda(), k.cuda(), v.cuda(), "1:2", block_mask=mask).cpu()
    got = dfss.dfss_attention_host(q, k, v, "1:2", block_mask=mask, chunks=4)
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    qf, kf, vf = (x.float() for x in (q, k, v))
    want = dfss.dfss_attention(qf.cuda(), kf.cuda(), vf.cuda(), "1:2", math_mode="tf32").cpu()
    got = dfss.dfss_attention_host(qf, kf, vf, "1:2", math_mode="tf32", chunks=3)
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    with pytest.raises(ValueError, match="host tensors"):
        dfss.dfss_attention_host(q.cuda(), k, v)


@pytest.mark.parametrize("case", range(8))
def test_block_mask_fuzz_many_items(case):
    """Randomised block masks on the fused kernels with several items per CTA: random tile
    sizes (multiples of 32, group-aligned), densities from very sparse to dense, 128-aligned
    block patterns and one-sided row bands; 2:4 / 1:2 / tf32 by case."""
    rng = np.random.default_rng(100 + case)
    n = int(rng.choice([256, 512, 768, 1024]))
    tr = int(rng.choice([32, 64, 128]))
    tc_ = int(rng.choice([32, 64, 128]))
    density = float(rng.choice([0.05, 0.3, 0.7, 0.95]))
    gr, gc = -(-n // tr), -(-n // tc_)
    style = case % 3
    if style == 0:      # i.i.d. tiles
        keep = rng.random((gr, gc)) < density
    elif style == 1:    # 128 x 128 blocks
        blk = rng.random((-(-n // 128), -(-n // 128))) < density
        keep = blk[(np.arange(gr) * tr) // 128][:, (np.arange(gc) * tc_) // 128]
    else:               # row bands: every other 128-row band keeps only a few key tiles
        keep = rng.random((gr, gc)) < density
        band = ((np.arange(gr) * tr) // 128) % 2 == 0
        keep[band] &= (np.arange(gc) * tc_ >= n - 128)[None, :]
    keep[np.arange(gr), rng.integers(0, gc, gr)] = True      # no empty row
    mask = dfss.BlockMask(keep, tr, tc_)
    mode, dt = [("2:4", torch.bfloat16), ("1:2", torch.float16), ("1:2", torch.float32)][case % 3]
    g = torch.Generator().manual_seed(200 + case)
    bh = max(2, 600 // (n // 256))                            # > 148 items: several per CTA
    q, k, v = (torch.randn((1, bh, n, 64), generator=g).to(dt).cuda() for _ in range(3))
    kw = {"math_mode": "tf32"} if dt == torch.float32 else {}
    out = _np(dfss.dfss_attention(q, k, v, mode, block_mask=mask, **kw))
    for h in (0, bh // 2, bh - 1):
        ops = [x[0, h].cpu().double().numpy() for x in (q, k, v)]
        if dt == torch.float32:
            ops = [_tf32(x) for x in ops]
        assert_close(out[0, h], _masked_oracle(*ops, mask, mode), 2e-2, 2e-2,
                     f"fuzz case {case}: n={n} tiles={tr}x{tc_} density={density} style={style} head {h}")


@pytest.mark.parametrize("shape", [(1, 64, 384), (2, 8, 1024), (1, 160, 512), (1, 2, 4096)])
def test_exact_fp32_3xtf32_matches_reference(shape):
    """Exact-FP32 1:2 attention with math "auto" on tcgen05 as 3xTF32: scores + selection
    (sddmm_tf32.cu), in-place row softmax, SpMM (spmm_tf32.cu).  Against the reference in float64
    at the 1e-5 bar (first and last heads, n <= 1024; 160 heads: several row blocks per CTA), and
    against the pure-FFMA mode ("ffma") everywhere within 5e-6 -- except rows whose selection
    differs at a near tie between the two fp32-accurate score computations (<= 1e-3 of the rows)."""
    b, h, n = shape
    (q, k, v), (q64, k64, v64) = seeded_qkv((b, h, n, 64), torch.float32, seed=n + h)
    out = _np(dfss.dfss_attention(q, k, v, "1:2"))
    for hh in (sorted({0, h - 1}) if n <= 1024 else []):
        sl = (slice(0, 1), slice(hh, hh + 1))
        assert_close(out[sl], oracle_attention(q64[sl], k64[sl], v64[sl], "1:2"), 1e-5, 1e-5,
                     f"3xtf32 {shape} h={hh}")
    ffma = _np(dfss.dfss_attention(q, k, v, "1:2", math_mode="ffma"))
    bad_rows = (np.abs(out - ffma) > 5e-6 + 5e-6 * np.abs(ffma)).any(axis=-1)
    assert bad_rows.sum() <= max(2, int(1e-3 * bad_rows.size)), (int(bad_rows.sum()), bad_rows.size)


def test_exact_fp32_3xtf32_unaligned_views_fall_back():
    """Views that are not 16-byte aligned take the FFMA pair instead of the 3xTF32 kernels (TMA /
    vector loads need alignment): same result as the aligned call within fp32 accuracy."""
    (q, k, v), _ = seeded_qkv((1, 64, 384, 64), torch.float32, seed=3)
    flat = [torch.empty(x.numel() + 1, device="cuda") for x in (q, k, v)]
    views = []
    for f, x in zip(flat, (q, k, v)):
        f[1:].copy_(x.reshape(-1))
        views.append(f[1:].view(x.shape))  # 4-byte offset
    assert views[0].data_ptr() % 16 != 0
    want = _np(dfss.dfss_attention(q, k, v, "1:2"))
    got = _np(dfss.dfss_attention(*views, "1:2"))
    bad_rows = (np.abs(got - want) > 5e-6 + 5e-6 * np.abs(want)).any(axis=-1)
    assert bad_rows.sum() <= 2


@pytest.mark.parametrize("n,mode,heads", [(512, "1:2", 3), (1024, "1:2", 3), (640, "2:4", 3), (384, "1:2", 64)])
def test_exact_fp32_longer_rows_match_reference(n, mode, heads):
    """Exact-FP32 path at the 1e-5 bar where the shared-memory-tiled SpMM runs (n >= 512, or
    >= 4 waves of 32-row blocks: 64 heads at n = 384; softmax fused), against the reference
    nm_attention in float64 (first, middle and last heads)."""
    (q, k, v), (q64, k64, v64) = seeded_qkv((1, heads, n, 64), torch.float32, seed=n + 7)
    out = _np(dfss.dfss_attention(q, k, v, mode, math_mode="ffma"))
    for h in sorted({0, heads // 2, heads - 1}):
        assert_close(out[:, h:h + 1], oracle_attention(q64[:, h:h + 1], k64[:, h:h + 1], v64[:, h:h + 1], mode),
                     1e-5, 1e-5, f"exact fp32 {mode} n={n} head {h}")
