"""Two processes running the CUDA path on one device: each rank computes its
floor + remainder shard of the flattened batch x heads with dfss_attention (bench.shard, the
same split bench.py --scaling strong uses), the shards are gathered through gloo on host copies,
and the result must equal the single-process output BITWISE -- heads are independent units,
so sharding changes nothing but where they run."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench

pytestmark = pytest.mark.gpu

CFG = dict(bench.CONFIGS["c2"], batch=1, heads=5, seq=512)  # 5 heads over 2 ranks: 3 + 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, q, mode):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import paper_2203_00091_b200 as dfss

    torch.cuda.set_device(0)
    total = CFG["batch"] * CFG["heads"]
    lo, hi = bench.shard(total, ws, rank)
    qkv = bench.make_inputs(CFG, lo, hi, "cuda")
    out = dfss.dfss_attention(qkv[0], qkv[1], qkv[2], mode).cpu()
    width = max(b - a for a, b in (bench.shard(total, ws, r) for r in range(ws)))
    pad = torch.zeros((width,) + tuple(out.shape[1:]), dtype=out.dtype)
    pad[: hi - lo] = out
    gathered = [torch.empty_like(pad) for _ in range(ws)]
    dist.all_gather(gathered, pad)
    if rank == 0:
        parts = [gathered[r][: bench.shard(total, ws, r)[1] - bench.shard(total, ws, r)[0]] for r in range(ws)]
        q.put(torch.cat(parts).float().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["2:4", "1:2"])
def test_two_ranks_on_one_device_equal_single_process(mode):
    import paper_2203_00091_b200 as dfss

    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q, mode)) for r in range(ws)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    total = CFG["batch"] * CFG["heads"]
    qkv = bench.make_inputs(CFG, 0, total, "cuda")
    want = dfss.dfss_attention(qkv[0], qkv[1], qkv[2], mode).float().cpu().numpy()
    assert got.shape == want.shape
    assert np.array_equal(got, want)
