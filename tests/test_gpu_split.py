"""GPU parity of the fused kernel's split last round (flash_tc.cu SplitPlan).

When bh * n / 256 items leave a partial last round on the persistent CTAs, those items are
cut along the keys into parts, each part leaves its unnormalised O / shift / row sum in the
workspace and the last part to finish merges them.  Outputs of the split items must match
the reference nm_attention (pipeline.py:15-32) like every other item: 2e-2 (bf16 / fp16).
"""

import numpy as np
import pytest
import torch

from gpu_helpers import assert_close, oracle_attention, seeded_qkv

import paper_2203_00091_b200 as dfss

pytestmark = pytest.mark.gpu


def _sms():
    return torch.cuda.get_device_properties(0).multi_processor_count


def _plan(bh, n, sms):
    items = bh * (n // 256)
    g = min(items, sms)
    rem = items % g
    parts = min(n // 128 // 4, g // rem) if rem else 1
    return items // g, rem, parts, g


def _last_round_heads(bh, n, sms):
    rounds, rem, parts, g = _plan(bh, n, sms)
    ipb = n // 256
    first_item = rounds * g
    return sorted({i // ipb for i in range(first_item, first_item + rem)})


@pytest.mark.parametrize("shape,dtype,mode", [
    ((1, 150, 1024, 64), torch.bfloat16, "2:4"),   # 600 items: rem 8, 2 parts of 4 tiles
    ((1, 37, 4096, 64), torch.float16, "2:4"),     # 592 items: no split (4 whole rounds)
    ((1, 38, 3072, 64), torch.float16, "2:4"),     # 456 items: rem 12, 6 uneven parts of 4 tiles
    ((1, 38, 3072, 64), torch.bfloat16, "1:2"),
    ((8, 12, 4096, 64), torch.bfloat16, "2:4"),    # config c4: rem 56, 2 parts of 16 tiles
])
def test_split_last_round_matches_reference(shape, dtype, mode):
    sms = _sms()
    bh, n = shape[0] * shape[1], shape[2]
    rounds, rem, parts, _ = _plan(bh, n, sms)
    if shape != (1, 37, 4096, 64):
        assert parts >= 2, "shape chosen so the last round is split on this GPU"
    (q, k, v), (q64, k64, v64) = seeded_qkv(shape, dtype, seed=11)
    out = dfss.dfss_attention(q, k, v, mode)
    heads = _last_round_heads(bh, n, sms)
    heads = sorted(set(heads[:6] + heads[-6:] + [0, bh // 2]))
    got = out.reshape(bh, n, 64)[heads].float().cpu().numpy()
    f = lambda x: x.reshape(bh, n, 64)[heads]  # noqa: E731
    want = oracle_attention(f(q64), f(k64), f(v64), mode)
    assert_close(got, want, 2e-2, 2e-2, f"split last round {shape} {mode} heads {heads}")


def test_split_repeated_calls_and_workspace_reuse():
    """The per-launch token tags the merge counters: back-to-back calls on one workspace (no
    memset in between) give the same output as fresh ones."""
    shape = (1, 150, 1024, 64)
    (q, k, v), _ = seeded_qkv(shape, torch.bfloat16, seed=2)
    need = dfss.workspace_bytes("2:4", q.dtype, 150, 1024, 64)
    assert need > 0
    ws = torch.full((need,), 0xAB, dtype=torch.uint8, device="cuda")  # garbage counters
    first = dfss.dfss_attention(q, k, v, "2:4", workspace=ws).clone()
    for _ in range(5):
        again = dfss.dfss_attention(q, k, v, "2:4", workspace=ws)
        assert torch.equal(again, first)
    fresh = dfss.dfss_attention(q, k, v, "2:4")
    assert torch.equal(fresh, first)
