"""Selection parity of the kernels that actually run.

The production path of nm_attention for 16-bit and tf32 inputs is a fused kernel that prunes
in registers (flash_tc.cu prune_exp_tile, flash_tf32.cu prune12_chunk).  Its DUMP build
(dfss_nm_attention_dump) stores the post-scale fp32 scores every prune compared and the
metadata words it handed to tcgen05.mma.sp.  Fed those same scores, the reference selection
(codec.py:104-123 / 289-313, _kernels_numba.py:145-184; restated in oracle/nmattn_oracle.py and
pinned to the reference by tests/test_oracle_golden.py) must produce the same nibbles and kept
masks BITWISE -- the contract of the reference's fused path (tests/test_fused.py:30-43,
acceptance c02).  Besides the bit-exact check, the kept-mask flips against the scores computed in
float64 from the same rounded inputs are counted and bounded (they measure fp32 accumulation,
not the selection rule).
"""

from __future__ import annotations

import zlib

import numpy as np
import pytest
import torch

from oracle import nmattn_oracle as ref

pytestmark = pytest.mark.gpu

dfss = pytest.importorskip("paper_2203_00091_b200")


def _kept_from_meta(meta: np.ndarray, mode: str) -> np.ndarray:
    """[rows, groups] logical nibbles -> kept bool [rows, cols] (codec.py:72-95)."""
    rows, groups = meta.shape
    if mode == "1:2":
        second = meta == 0xE
        kept = np.stack((~second, second), axis=2)
        return kept.reshape(rows, 2 * groups)
    lo, hi = meta & 3, (meta >> 2) & 3
    kept = np.zeros((rows, groups, 4), dtype=bool)
    np.put_along_axis(kept, lo[..., None].astype(np.int64), True, axis=2)
    np.put_along_axis(kept, hi[..., None].astype(np.int64), True, axis=2)
    return kept.reshape(rows, 4 * groups)


def _check_heads(dump, q64, k64, mode: str, heads, present=None, flip_budget=1e-4, what=""):
    """Bit-exact nibbles / kept masks vs the reference selection on the dumped scores, for the
    flattened (batch, head) indices `heads`; flips vs float64 scores counted and bounded."""
    n = dump.scores.shape[-1]
    gs = 2 if mode == "1:2" else 4
    scores = dump.scores.reshape(-1, n, n)
    meta = dump.meta.reshape(-1, n, n // gs)
    qf, kf = q64.reshape(-1, n, q64.shape[-1]), k64.reshape(-1, n, k64.shape[-1])
    scale = 1.0 / np.sqrt(q64.shape[-1])
    flips = groups = 0
    for h in heads:
        s = scores[h].double().cpu().numpy()
        m = meta[h].cpu().numpy()
        gmask = np.ones((n, n // gs), dtype=bool) if present is None else present[:, ::gs]
        assert np.isfinite(s[np.repeat(gmask, gs, axis=1)]).all(), f"{what} head {h}: prune read non-finite scores"
        s_fill = np.where(np.isfinite(s), s, 0.0)
        kept_ref, _, nib_ref = ref.select_rows(s_fill, mode)
        bad = (m != nib_ref) & gmask
        if bad.any():
            r, g = np.argwhere(bad)[0]
            raise AssertionError(
                f"{what} head {h}: {int(bad.sum())} / {int(gmask.sum())} nibbles differ from the reference "
                f"selection on the same scores; first at row {r} group {g}: gpu 0x{m[r, g]:x} ref 0x{nib_ref[r, g]:x} "
                f"scores {s[r, gs * g:gs * g + gs].tolist()}")
        kmask = np.repeat(gmask, gs, axis=1)
        assert np.array_equal(_kept_from_meta(m, mode)[kmask], kept_ref[kmask]), f"{what} head {h}: kept mask"
        # end-to-end flips: the same rounded inputs scored in float64 (the reference's arithmetic)
        s64 = (qf[h] @ kf[h].T) * scale
        _, _, nib64 = ref.select_rows(s64, mode)
        flips += int(((nib64 != m) & gmask).sum())
        groups += int(gmask.sum())
    assert flips <= flip_budget * groups, f"{what}: {flips} / {groups} kept-mask flips vs float64 scores"
    return flips, groups


def _inputs(shape, dtype, seed=0, kind="normal"):
    g = torch.Generator().manual_seed(seed)
    if kind == "normal":
        x = [torch.randn(shape, generator=g) for _ in range(3)]
    elif kind == "lattice":
        # small integers: exact fp32 products and sums, so scores tie exactly and often
        x = [torch.randint(-2, 3, shape, generator=g).float() for _ in range(3)]
    elif kind == "zeros":
        # rows of +0 and -0 queries: every score of those rows is a signed zero, all tied
        x = [torch.randn(shape, generator=g) for _ in range(3)]
        x[0][..., ::3, :] = 0.0
        x[0][..., 1::3, :] = -0.0
    else:
        raise ValueError(kind)
    x = [t.to(dtype) for t in x]
    return [t.cuda() for t in x], [t.double().numpy() for t in x]


CASES = [
    # (mode, dtype, math, shape, kind, path): production head shapes and kernels
    ("2:4", torch.bfloat16, "auto", (2, 3, 512, 64), "normal", "fused-16bit"),        # c2 heads, two-set kernel
    ("2:4", torch.float16, "auto", (1, 4, 1024, 64), "normal", "fused-16bit"),        # c3 heads
    ("2:4", torch.bfloat16, "auto", (1, 2, 4096, 64), "normal", "fused-16bit"),       # c4 heads
    ("2:4", torch.bfloat16, "auto", (1, 3, 384, 64), "normal", "fused-16bit"),        # one-set kernel (n % 256)
    ("1:2", torch.bfloat16, "auto", (2, 3, 512, 64), "normal", "fused-16bit"),        # 1:2 as the 2:4 pattern
    ("1:2", torch.float16, "auto", (1, 3, 640, 64), "normal", "fused-16bit"),         # one-set, 1:2
    ("1:2", torch.float32, "tf32", (2, 3, 512, 64), "normal", "fused-tf32"),          # configs[4] 1:2 tf32
    ("1:2", torch.float32, "tf32", (1, 3, 384, 64), "normal", "fused-tf32"),          # empty half of last block
    ("2:4", torch.bfloat16, "auto", (1, 4, 512, 64), "lattice", "fused-16bit"),       # exact ties
    ("1:2", torch.bfloat16, "auto", (1, 4, 512, 64), "lattice", "fused-16bit"),
    ("1:2", torch.float32, "tf32", (1, 4, 512, 64), "lattice", "fused-tf32"),
    ("2:4", torch.float16, "auto", (1, 4, 384, 64), "lattice", "fused-16bit"),
    ("2:4", torch.bfloat16, "auto", (1, 4, 512, 64), "zeros", "fused-16bit"),         # +-0 queries
    ("1:2", torch.float16, "auto", (1, 4, 512, 64), "zeros", "fused-16bit"),
    ("1:2", torch.float32, "tf32", (1, 4, 512, 64), "zeros", "fused-tf32"),
    # staged paths through the same hook
    ("2:4", torch.float32, "auto", (1, 12, 384, 64), "normal", "staged-ffma"),        # c1-shaped (2:4 here)
    ("1:2", torch.float32, "ffma", (1, 12, 384, 64), "normal", "staged-ffma"),        # c1, pure FFMA
    ("1:2", torch.float32, "auto", (1, 12, 384, 64), "normal", "staged-3xtf32"),      # c1 (3xTF32 on tcgen05)
    ("1:2", torch.float32, "auto", (1, 8, 512, 64), "lattice", "staged-3xtf32"),      # exact ties, 3xTF32
    ("1:2", torch.float32, "auto", (1, 8, 512, 64), "zeros", "staged-3xtf32"),        # +-0 queries, 3xTF32
]


@pytest.mark.parametrize("mode,dtype,math_mode,shape,kind,path", CASES,
                         ids=[f"{c[0]}-{str(c[1]).split('.')[-1]}-{c[2]}-{c[3][-2]}-{c[4]}" for c in CASES])
def test_kernel_selection_bitexact_on_dumped_scores(mode, dtype, math_mode, shape, kind, path):
    (q, k, v), (q64, k64, _) = _inputs(shape, dtype, seed=zlib.crc32(repr((mode, kind, shape)).encode()) & 0xFFFF, kind=kind)
    if math_mode == "tf32":  # the tf32 MMA reads fp32 operands truncated to tf32
        q64, k64 = (np.frombuffer((x.astype(np.float32).view(np.uint32) & 0xFFFFE000).tobytes(),
                                  dtype=np.float32).reshape(x.shape).astype(np.float64) for x in (q64, k64))
    dump = dfss.dfss_attention_dump(q, k, v, mode, math_mode=math_mode)
    assert dump.path == path
    # the dump build computes the same output as the production kernel
    ref_out = dfss.dfss_attention(q, k, v, mode, math_mode=math_mode)
    torch.cuda.synchronize()
    assert torch.equal(dump.out, ref_out), "DUMP instantiation changed the output"
    bh = int(np.prod(shape[:-2]))
    # tf32: truncation differs from the MMA's internal tf32 conversion on ties only in rounding
    # mode; the selection itself is compared on the dumped scores, the flip count is a report
    budget = 2e-2 if math_mode == "tf32" else 1e-4
    _check_heads(dump, q64, k64, mode, range(bh), flip_budget=budget, what=f"{path} {mode} {kind}")


def _heads_over_rounds(bh: int, items_per_head: int, sms: int = 148):
    """Heads whose items land in the first, middle and last persistent-CTA rounds."""
    items = bh * items_per_head
    picks = {0, bh - 1}
    for rnd in range(0, (items + sms - 1) // sms):
        picks.add(min(bh - 1, (rnd * sms) // items_per_head))
        picks.add(min(bh - 1, (rnd * sms + sms - 1) // items_per_head))
    return sorted(picks)


@pytest.mark.parametrize("cfg", ["c2", "c4"])
def test_production_shape_selection_bitexact(cfg):
    """Full BASELINE shapes (every persistent-CTA round, deferred epilogues, barrier phases
    carried across items): selection bit-exact on the dumped scores of heads from every round."""
    shape, dtype = {"c2": ((32, 12, 512, 64), torch.bfloat16), "c4": ((8, 12, 4096, 64), torch.bfloat16)}[cfg]
    (q, k, v), (q64, k64, _) = _inputs(shape, dtype, seed=7)
    dump = dfss.dfss_attention_dump(q, k, v, "2:4")
    assert dump.path == "fused-16bit"
    n = shape[-2]
    heads = _heads_over_rounds(shape[0] * shape[1], n // 256)
    if cfg == "c4":
        heads = [heads[0], heads[len(heads) // 2], heads[-1]]
    _check_heads(dump, q64, k64, "2:4", heads, what=cfg)


def test_block_masked_selection_bitexact():
    """Masked fused kernel: chunks in masked tiles carry no selection; every present group's
    nibble equals the reference selection on the dumped scores (fused.py:73-82)."""
    n = 1024
    (q, k, v), (q64, k64, _) = _inputs((1, 4, n, 64), torch.bfloat16, seed=3)
    rng = np.random.default_rng(5)
    keep = rng.random((n // 64, n // 64)) < 0.6
    keep[np.arange(n // 64), np.arange(n // 64)] = True  # no empty row
    mask = dfss.BlockMask(keep, 64, 64)
    for mode in ("2:4", "1:2"):
        dump = dfss.dfss_attention_dump(q, k, v, mode, block_mask=mask)
        assert dump.path == "fused-16bit"
        present = mask.dense_keep(n, n)
        _check_heads(dump, q64, k64, mode, range(4), present=present, what=f"masked {mode}")
        gs = 2 if mode == "1:2" else 4
        absent = ~present[:, ::gs]
        # nothing selected there: 0 (skipped step / absent pair) or the 0x4 padding nibble (2:4)
        vals = dump.meta.reshape(-1, n, n // gs).cpu().numpy()[:, absent]
        assert np.isin(vals, [0, 0x4] if mode == "2:4" else [0]).all()
