"""CPU-only checks of the drop-in boundary: the C-ABI library loads, exports
exactly what include/dfss.h declares, and the host layer validates like the
reference (same ValueError fragments) before touching a device."""

import os
import re

import numpy as np
import pytest
import torch

from conftest import ROOT, golden

import paper_2203_00091_b200 as dfss
from paper_2203_00091_b200 import _lib
from paper_2203_00091_b200.fused import FusedStats, _stats


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "dfss.h")).read()
    return sorted(set(re.findall(r"\b(dfss_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _declared_symbols()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(lib, name), name
    # the ctypes signature table covers the header exactly
    assert sorted(_lib.SIGNATURES) == declared
    assert lib.dfss_version() >= 100


def test_meta_hw_geometry():
    lib = _lib.load()
    # n^2/8 bytes per head when aligned (2:4: 4 bits per 4 scores; 1:2: 4 bits per 2)
    assert lib.dfss_meta_hw_words(4, 1, 512, 512) * 4 == 512 * 512 // 8
    assert lib.dfss_meta_hw_words(2, 1, 384, 384) * 4 == 384 * 384 // 4
    # padding to 128 rows and 8-group chunks
    assert lib.dfss_meta_hw_words(4, 3, 100, 36) == 3 * 1 * 2 * 128
    assert lib.dfss_meta_hw_words(7, 1, 4, 4) == -1


def test_status_strings():
    lib = _lib.load()
    assert lib.dfss_status_string(0) == b"ok"
    assert lib.dfss_status_string(-1) == b"invalid argument"


def test_c_abi_validation_rejects_before_launch():
    lib = _lib.load()
    # bad mode, misaligned columns, null pointers: all DFSS_ERR_INVALID without a device
    assert lib.dfss_sddmm_prune(None, None, None, None, 1.0, 3, 0, 0, 0, 1, 8, 8, 4, None, 0, 0, None, None, None) == -1
    assert lib.dfss_sddmm_prune(None, None, None, None, 1.0, 4, 0, 0, 0, 1, 8, 6, 4, None, 0, 0, None, None, None) == -1
    assert b"group-aligned" in lib.dfss_last_error()
    assert lib.dfss_spmm(None, None, None, None, 2, 0, 0, 0, 1, 4, 4, 2, None, 0, 0, None, None) == -1
    assert lib.dfss_nm_attention_workspace_bytes(4, 1, 2, 512, 64) >= 2 * 512 * 256 * 2 + 2 * 512 * 512 // 8


def test_host_validation_messages_match_reference():
    q = torch.zeros(5, 4)
    k = torch.zeros(5, 4)
    with pytest.raises(ValueError, match="group-aligned"):
        dfss.sddmm_prune(q, k, dfss.SparsityMode.ONE_OF_TWO, 1.0)
    with pytest.raises(ValueError, match="shape mismatch"):
        dfss.sddmm_prune(q, torch.zeros(4, 3), dfss.SparsityMode.ONE_OF_TWO, 1.0)
    q64 = torch.zeros(64, 4)
    bad_grid = dfss.BlockMask(np.ones((3, 1), dtype=bool), tile_rows=32, tile_cols=64)
    with pytest.raises(ValueError, match="grid"):
        dfss.sddmm_prune(q64, q64, dfss.SparsityMode.ONE_OF_TWO, 1.0, bad_grid)
    wrong_tiles = dfss.BlockMask(np.ones((2, 1), dtype=bool), tile_rows=32, tile_cols=128)
    with pytest.raises(ValueError, match="tiling"):
        dfss.sddmm_prune(q64, q64, dfss.SparsityMode.ONE_OF_TWO, 1.0, wrong_tiles)
    with pytest.raises(ValueError, match="CUDA"):
        dfss.sddmm_prune(q64, q64, dfss.SparsityMode.ONE_OF_TWO, 1.0)
    with pytest.raises(ValueError, match="dense"):
        FusedStats(peak_tile_elems=1, dense_elems_written=3, nonzeros_written=0, nibbles_written=0)
    with pytest.raises(ValueError, match="unknown sparsity mode"):
        dfss.SparsityMode.parse("3:4")
    with pytest.raises(ValueError, match="malformed nibble"):
        dfss.slots_for_nibble(0x0)
    with pytest.raises(ValueError, match="shape"):
        dfss.dfss_attention(torch.zeros(8, 4), torch.zeros(8, 4), torch.zeros(6, 4))


def test_backend_is_single_and_fixed():
    assert dfss.active_backend() == "cuda-sm100a"
    for name in ("numba", "numpy"):
        with pytest.raises(ValueError, match="no CPU fallback"):
            dfss.set_backend(name)


def test_fused_stats_match_reference_counters():
    g = golden("fused.npz")
    st = _stats(4, 4, 2, 32, 64, None)
    assert [st.peak_tile_elems, st.nonzeros_written, st.nibbles_written] == list(g["identity_stats"])
    for i in range(int(g["n_cases"])):
        mode = str(g[f"case{i}_mode"])
        n, m = g[f"case{i}_q"].shape[0], g[f"case{i}_k"].shape[0]
        st = _stats(n, m, 2 if mode == "1:2" else 4, 32, 64, None)
        assert [st.peak_tile_elems, st.nonzeros_written, st.nibbles_written] == list(g[f"case{i}_stats"]), i
    st = _stats(64, 64, 2, 32, 32, g["masked_keep"])
    assert [st.peak_tile_elems, st.nonzeros_written, st.nibbles_written] == list(g["masked_stats"])


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2203_00091_b200")
    pat = re.compile(r"^\s*(from\s+oracle|import\s+oracle)|liboracle|nmattn_oracle", re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                assert not pat.search(open(os.path.join(dirpath, f)).read()), f


def test_container_header_validation_and_nibble_packing():
    """NMCS parsing rejects malformed headers before touching the GPU (container.py:74-92);
    nibble packing is the reference's (low nibble first, zero pad)."""
    import struct

    import numpy as np

    from conftest import golden
    from paper_2203_00091_b200 import container

    g = golden("container.npz")
    raw = g["nmcs_24"].tobytes()
    with pytest.raises(ValueError, match="truncated"):
        container.from_bytes(raw[:10])
    with pytest.raises(ValueError, match="bad magic"):
        container.from_bytes(b"XXXX" + raw[4:])
    with pytest.raises(ValueError, match="unsupported container version"):
        container.from_bytes(raw[:4] + bytes([2]) + raw[5:])
    with pytest.raises(ValueError, match="unknown mode code"):
        container.from_bytes(raw[:5] + bytes([7]) + raw[6:])
    with pytest.raises(ValueError, match="container size"):
        container.from_bytes(raw + b"\0")
    magic, version, mode, layout, rows, cols = struct.unpack_from("<4sBBBII", raw)
    assert (magic, version, mode, layout, rows, cols) == (b"NMCS", 1, 2, 0, 33, 64)
    nib = np.array([4, 8, 9, 0xC, 0xD], dtype=np.uint8)
    packed = container.pack_nibbles(nib)
    assert packed == bytes([0x84, 0xC9, 0x0D])
    assert (container.unpack_nibbles(packed, 5) == nib).all()
    # the golden file's nibble section is exactly the reference packing of its own stream
    nz_end = 15 + 8 * rows * cols // 2
    stream = container.unpack_nibbles(raw[nz_end:], rows * cols // 4)
    assert container.pack_nibbles(stream) == raw[nz_end:]
