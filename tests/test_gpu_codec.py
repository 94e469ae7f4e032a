"""GPU decode paths of the codec against the reference (nonzero_columns,
decompress, codec.py:346-372), fed the reference-written compressed matrices of
tests/golden/codec.npz and fused.npz."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import golden
from oracle import nmattn_oracle as ref

pytestmark = pytest.mark.gpu

dfss = pytest.importorskip("paper_2203_00091_b200")


@pytest.mark.parametrize("mode", ["1:2", "2:4"])
def test_nonzero_columns_and_decompress_match_reference(mode):
    g = golden("codec.npz")
    key = mode.replace(":", "")
    for i in range(int(g["n_scores"])):
        s = g[f"scores{i}"]
        rows, cols = s.shape
        nz, meta = g[f"scores{i}_{key}_nonzeros"], g[f"scores{i}_{key}_metadata"]
        c = dfss.CompressedSparse.from_logical(rows, cols, mode, torch.from_numpy(nz).cuda(), torch.from_numpy(meta))
        got_cols = dfss.nonzero_columns(c).cpu().numpy()
        assert got_cols.dtype == np.int64
        assert np.array_equal(got_cols, ref.nonzero_columns(meta, rows, cols, mode)), f"scores{i} columns"
        dense = dfss.decompress(c).data.cpu().numpy()
        # decompress(compress_logical(s)) == prune_dense(s) (codec.py:324-372), bitwise in float64
        assert np.array_equal(dense, np.where(g[f"scores{i}_{key}_mask"], s, 0.0)), f"scores{i} decompress"
        assert np.array_equal(dense, ref.decompress(nz, meta, cols, mode))
        # round trip of the logical stream through the tcgen05 word layout
        assert np.array_equal(c.metadata.cpu().numpy(), meta)


def test_masked_decode_matches_reference_fused_output():
    """Masked tiles are structurally absent (codec.py:150-200): their columns decode to -1 and
    decompress leaves them zero; present entries decode like the reference."""
    g = golden("fused.npz")
    nz, meta, keep = g["masked_nonzeros"], g["masked_metadata"], g["masked_keep"]
    rows, cols = 64, 64
    mask = dfss.BlockMask(keep, 32, 32)
    c = dfss.CompressedSparse.from_logical(rows, cols, "1:2", torch.from_numpy(nz).cuda(), torch.from_numpy(meta),
                                           block_mask=mask)
    got = dfss.nonzero_columns(c).cpu().numpy()
    present = mask.nonzero_keep(rows, cols)
    want = ref.nonzero_columns(meta, rows, cols, "1:2")
    assert np.array_equal(got[present], want[present]) and (got[~present] == -1).all()
    dense = dfss.decompress(c).data.cpu().numpy()
    assert np.array_equal(dense, ref.decompress(nz, meta, cols, "1:2") * mask.dense_keep(rows, cols))
    assert np.array_equal(c.metadata.cpu().numpy(), meta)  # zero filler in masked tiles, as the reference
