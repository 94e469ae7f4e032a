"""Generate golden vectors for the DFSS hot path from the REAL reference.

Run in the build container, where the reference package is importable:

    PYTHONPATH=/root/reference/pkg/src NMATTN_BACKEND=numba \
        python tests/golden/make_golden.py

Every array written here is an output of ``nmattn`` 0.1.0 itself (numba
backend, the reference default, backend.py:32-42) on seeded inputs.  The
fixtures pin the CPU oracle (oracle/) that the GPU tests use as the checker
on the GPU box, where /root/reference does not exist.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    import nmattn
    from nmattn import (
        AttentionInputs,
        BlockMask,
        DenseMatrix,
        SparsityMode,
        compress_logical,
        full_attention,
        gemm_scaled,
        nm_attention,
        prune_dense,
        sddmm_prune,
        select_group,
        softmax_rows,
        spmm,
    )

    nmattn.set_backend("numba")
    modes = {"1:2": SparsityMode.ONE_OF_TWO, "2:4": SparsityMode.TWO_OF_FOUR}
    out: dict[str, np.ndarray] = {}

    # ---- select_group anchors (test_codec.py:37-63) + the fp32 sum-tie counter-example
    groups = [
        ("1:2", [3.0, -5.0]), ("1:2", [-5.0, 3.0]), ("1:2", [1.0, 1.0]), ("1:2", [-0.0, 0.0]),
        ("2:4", [0.5, -1.2, 2.0, 0.1]), ("2:4", [1.0, 1.0, 1.0, 1.0]), ("2:4", [0.0, -0.0, 0.0, -0.0]),
        ("2:4", [-1.0, -2.0, -3.0, -4.0]), ("2:4", [-4.0, -3.0, -2.0, -1.0]), ("2:4", [2.0, 1.0, 2.0, 1.0]),
        ("2:4", [1000.0, np.float32(1e-5), np.float32(2e-5), -3.0]), ("2:4", [1.0, 2.0, 2.0, 2.0]),
        ("2:4", [5.0, 5.0, 7.0, 5.0]),
    ]
    for i, (mode, vals) in enumerate(groups):
        sel = select_group(np.asarray(vals, dtype=np.float64), modes[mode])
        out[f"group{i}_mode"] = np.array(mode)
        out[f"group{i}_values"] = np.asarray(vals, dtype=np.float64)
        out[f"group{i}_kept"] = np.asarray(sel.kept, dtype=np.int64)
        out[f"group{i}_nibble"] = np.array(sel.nibble, dtype=np.uint8)
    out["n_groups"] = np.array(len(groups))

    # ---- score matrices -> compress_logical / prune_dense (the metadata + mask oracle)
    rng = np.random.default_rng(20261017)
    score_cases = []
    score_cases.append(rng.standard_normal((32, 64)))
    score_cases.append(rng.integers(-2, 3, size=(32, 64)).astype(float))  # heavy ties
    sz = np.zeros((8, 32))
    sz[::2, 1::2] = -0.0
    sz[1::2, ::3] = 0.0
    score_cases.append(sz)  # signed zeros
    bf = rng.standard_normal((64, 128)).astype(np.float32)
    bf = (bf.view(np.uint32) & 0xFFFF0000).view(np.float32).astype(np.float64)  # bf16-rounded: many near ties
    score_cases.append(bf)
    ce = np.tile(np.array([1000.0, np.float32(1e-5), np.float32(2e-5), -3.0]), (4, 8))
    score_cases.append(ce)
    score_cases.append((rng.standard_normal((128, 256)) * 8).astype(np.float32).astype(np.float64))
    for i, s in enumerate(score_cases):
        for mode in ("1:2", "2:4"):
            c = compress_logical(DenseMatrix(s), modes[mode])
            _, mask = prune_dense(DenseMatrix(s), modes[mode])
            key = f"scores{i}_{mode.replace(':', '')}"
            out[f"{key}_nonzeros"] = c.nonzeros
            out[f"{key}_metadata"] = c.metadata
            out[f"{key}_mask"] = mask.bits
        out[f"scores{i}"] = s
    out["n_scores"] = np.array(len(score_cases))
    np.savez_compressed(os.path.join(HERE, "codec.npz"), **out)

    # ---- fused sddmm_prune instances (test_fused.py:18-63, test_acceptance.py:90-104)
    out = {}
    eye = DenseMatrix(np.eye(4))
    c, st = sddmm_prune(eye, eye, modes["1:2"], 1.0)
    out["identity_nonzeros"] = c.nonzeros
    out["identity_metadata"] = c.metadata
    out["identity_stats"] = np.array([st.peak_tile_elems, st.nonzeros_written, st.nibbles_written])
    rng = np.random.default_rng(202)
    cases = []
    for i in range(24):
        mode = "1:2" if i % 2 == 0 else "2:4"
        n = int(rng.choice([4, 16, 32, 48, 64, 96])) * (2 if mode == "2:4" else 1)
        m = n if i % 3 else n + 4 * int(rng.integers(1, 5))
        d = int(rng.integers(1, 24))
        scale = float(rng.standard_normal()) or 1.0
        if i % 5 == 4:
            q = rng.integers(-1, 2, size=(n, d)).astype(float)
            kk = rng.integers(-1, 2, size=(m, d)).astype(float)
        else:
            q = rng.standard_normal((n, d))
            kk = rng.standard_normal((m, d))
        fc, st = sddmm_prune(DenseMatrix(q), DenseMatrix(kk), modes[mode], scale)
        out[f"case{i}_mode"] = np.array(mode)
        out[f"case{i}_q"] = q
        out[f"case{i}_k"] = kk
        out[f"case{i}_scale"] = np.array(scale)
        out[f"case{i}_nonzeros"] = fc.nonzeros
        out[f"case{i}_metadata"] = fc.metadata
        out[f"case{i}_stats"] = np.array([st.peak_tile_elems, st.nonzeros_written, st.nibbles_written])
        cases.append(i)
    # block-masked fused case (test_fused.py:66-82)
    q = rng.standard_normal((64, 12))
    kk = rng.standard_normal((64, 12))
    keep = np.array([[True, False], [True, True]])
    fc, st = sddmm_prune(DenseMatrix(q), DenseMatrix(kk), modes["1:2"], 1.0,
                         BlockMask(keep, tile_rows=32, tile_cols=32), tile_rows=32, tile_cols=32)
    out["masked_q"], out["masked_k"], out["masked_keep"] = q, kk, keep
    out["masked_nonzeros"], out["masked_metadata"] = fc.nonzeros, fc.metadata
    out["masked_stats"] = np.array([st.peak_tile_elems, st.nonzeros_written, st.nibbles_written])
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "fused.npz"), **out)

    # ---- softmax_rows and spmm (test_sparse_ops.py)
    out = {}
    rng = np.random.default_rng(303)
    for i in range(8):
        mode = "1:2" if i % 2 == 0 else "2:4"
        rows, cols = 4 * int(rng.integers(1, 9)), 8 * int(rng.integers(1, 9))
        s = rng.standard_normal((rows, cols)) * (10.0 if i % 3 == 0 else 1.0)
        if i == 5:
            s += 1000.0
        c = compress_logical(DenseMatrix(s), modes[mode])
        sm = softmax_rows(c)
        v = rng.standard_normal((cols, int(rng.integers(1, 20))))
        o = spmm(sm, DenseMatrix(v))
        out[f"case{i}_mode"] = np.array(mode)
        out[f"case{i}_nonzeros"] = c.nonzeros
        out[f"case{i}_metadata"] = c.metadata
        out[f"case{i}_dense_cols"] = np.array(cols)
        out[f"case{i}_softmax"] = sm.nonzeros
        out[f"case{i}_v"] = v
        out[f"case{i}_spmm"] = o.data
    out["n_cases"] = np.array(8)
    np.savez_compressed(os.path.join(HERE, "sparse_ops.npz"), **out)

    # ---- end-to-end nm_attention / full_attention
    out = {}
    rng = np.random.default_rng(20240101)
    q, k, v = (rng.standard_normal((256, 64)) for _ in range(3))
    inputs = AttentionInputs(DenseMatrix(q), DenseMatrix(k), DenseMatrix(v))
    out["pin_q"], out["pin_k"], out["pin_v"] = q, k, v
    out["pin_nm12"] = nm_attention(inputs, modes["1:2"]).data
    out["pin_nm24"] = nm_attention(inputs, modes["2:4"]).data
    out["pin_full"] = full_attention(inputs).data
    rng = np.random.default_rng(7)
    for i, (n, d) in enumerate([(64, 16), (128, 64), (96, 8)]):
        q, k, v = (rng.standard_normal((n, d)) for _ in range(3))
        inputs = AttentionInputs(DenseMatrix(q), DenseMatrix(k), DenseMatrix(v))
        out[f"case{i}_q"], out[f"case{i}_k"], out[f"case{i}_v"] = q, k, v
        for mode in ("1:2", "2:4"):
            out[f"case{i}_nm{mode.replace(':', '')}"] = nm_attention(inputs, modes[mode]).data
            scores = gemm_scaled(inputs.q, inputs.k, 1.0 / math.sqrt(d))
            cs = compress_logical(scores, modes[mode])
            out[f"case{i}_meta{mode.replace(':', '')}"] = cs.metadata
    out["n_cases"] = np.array(3)
    np.savez_compressed(os.path.join(HERE, "pipeline.npz"), **out)
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    sys.exit(main())
