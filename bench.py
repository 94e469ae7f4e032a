#!/usr/bin/env python3
"""DFSS attention benchmark on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dfss|reference] [--config c2]
                    [--scaling weak|strong]

A step is one DFSS attention pass (dfss_attention: for 16-bit inputs ONE fused kernel --
QK^T on tcgen05 -> 2:4 / 1:2 prune in registers -> exp -> tcgen05.mma.sp P.V) over this rank's
shard of the flattened batch x heads, synthetic N(0,1) Q/K/V resident in HBM (L2 flushed
between timed steps).  Sharding: batch x heads are independent units with no data exchange
(SURVEY §8(e)).  --scaling weak (default): every rank owns the config's B*H heads, the job's
global batch is N x B.  --scaling strong: the config's B*H heads are split over the N ranks,
floor + remainder (c1: 12 heads on 8 ranks -> 2,2,2,2,1,1,1,1).  Inputs are seeded per
(seed, global head), so a rank's shard equals the same slice of a 1-GPU run.  The compute phase
has no collective; one NCCL all-gather of the output shards after the timed region is the
end-to-end check.  Rank 0 prints ONE JSON line; numbers taken under a profiler are never
reported.  --impl reference times the reference's CPU algorithm (oracle/dfss_oracle.c, the C
restatement of nmattn.nm_attention, bitwise equal to the numba reference on the golden
fixtures) on the host cores, on the same config keys.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

#: BASELINE.json configs; c2 (configs[1]) is the one the metric is quoted on at N=1
CONFIGS = {
    "c1": dict(batch=1, heads=12, seq=384, d=64, mode="1:2", dtype="float32",
               desc="DFSS 1:2 fp32 attention, batch 1, 12 heads, seq 384, head_dim 64"),
    "c2": dict(batch=32, heads=12, seq=512, d=64, mode="2:4", dtype="bfloat16",
               desc="BERT-base-shaped DFSS 2:4 bf16 attention, batch 32, 12 heads, seq 512, head_dim 64"),
    "c3": dict(batch=16, heads=16, seq=1024, d=64, mode="2:4", dtype="float16",
               desc="BERT-large-shaped DFSS 2:4 fp16 attention, batch 16, 16 heads, seq 1024, head_dim 64"),
    "c4": dict(batch=8, heads=12, seq=4096, d=64, mode="2:4", dtype="bfloat16",
               desc="Long-sequence DFSS 2:4 bf16 attention, batch 8, 12 heads, seq 4096, head_dim 64"),
}
# configs[4]: the sequence sweep, batch 8 x 12 heads (SURVEY §8(d) proposal), reported in the
# default line's "sweep" object: 2:4 bf16 and 1:2 bf16 (fused kernel), 1:2 tf32 (fused tf32
# kernel) and, for reference, 1:2 exact FP32 (staged FFMA kernels)
for _n in (384, 512, 768, 1024, 2048, 4096):
    CONFIGS[f"c5_24_{_n}"] = dict(batch=8, heads=12, seq=_n, d=64, mode="2:4", dtype="bfloat16",
                                  desc=f"sweep 2:4 bf16, batch 8, 12 heads, seq {_n}")
    CONFIGS[f"c5_12_{_n}"] = dict(batch=8, heads=12, seq=_n, d=64, mode="1:2", dtype="bfloat16",
                                  desc=f"sweep 1:2 bf16, batch 8, 12 heads, seq {_n}")
    CONFIGS[f"c5_12tf32_{_n}"] = dict(batch=8, heads=12, seq=_n, d=64, mode="1:2", dtype="float32", math="tf32",
                                      desc=f"sweep 1:2 tf32 (fp32 inputs), batch 8, 12 heads, seq {_n}")
    if _n <= 1024:
        CONFIGS[f"c5_12f32_{_n}"] = dict(batch=8, heads=12, seq=_n, d=64, mode="1:2", dtype="float32",
                                         desc=f"sweep 1:2 fp32 (fp32-accurate: 3xTF32 on tcgen05 from ~1 M scores, FFMA below), batch 8, 12 heads, seq {_n}")
DT = {"float32": torch.float32, "bfloat16": torch.bfloat16, "float16": torch.float16}
DTYPE_TAG = {"float32": "f32", "bfloat16": "bf16", "float16": "f16"}
METRIC = "DFSS attention ms & speedup vs dense attention (seq 512–4096) on B200; TFLOPS"
UNIT = "TFLOP/s (dense-equivalent 4*n^2*d per head)"
L2_FLUSH_BYTES = 256 << 20
#: nominal B200 FP32 FFMA peak (148 SMs x 128 FMA/clk x 2 x 1.965 GHz): not in MEASURED_PEAKS.json
FP32_FFMA_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(d.get("sm_max_mhz", 1965.0)), "measured"
    return 6650.0, 1590.0, 1965.0, "fallback (B200_PROFILING.md)"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def shard(total: int, ws: int, rank: int):
    """Contiguous floor + remainder split of `total` units over `ws` ranks: the first
    total % ws ranks own one extra unit (12 over 8 -> 2,2,2,2,1,1,1,1)."""
    base, rem = divmod(total, ws)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def job_heads(cfg, ws: int, scaling: str) -> int:
    """Global batch x heads of the job: weak scaling multiplies the config by the rank count."""
    per = cfg["batch"] * cfg["heads"]
    return per * ws if scaling == "weak" else per


def make_inputs(cfg, lo, hi, device, seed=0):
    """Per-head seeded inputs (seed, global head index): shards equal the 1-GPU run."""
    n, d = cfg["seq"], cfg["d"]
    dt = DT[cfg["dtype"]]
    qkv = torch.empty((3, hi - lo, n, d), dtype=dt)
    for i, h in enumerate(range(lo, hi)):
        g = torch.Generator().manual_seed(seed * 1_000_003 + h)
        qkv[:, i] = torch.randn((3, n, d), generator=g, dtype=torch.float32).to(dt)
    return qkv.to(device)


def config_block(cfg_name: str, ws: int, scaling: str, heads_per_rank) -> dict:
    """The `config` object of both arms (key-identical, so the driver can pair them)."""
    cfg = CONFIGS[cfg_name]
    total = job_heads(cfg, ws, scaling)
    return {"workload": f"{cfg_name}: {cfg['desc']}", "batch": cfg["batch"], "heads": cfg["heads"],
            "seq_len": cfg["seq"], "head_dim": cfg["d"], "mode": cfg["mode"],
            "math": cfg.get("math", "auto"), "global_batch": total // cfg["heads"], "global_heads": total,
            "parallelism": f"bh-shard{ws}", "scaling": scaling, "heads_per_rank": heads_per_rank,
            "l2": "flushed between timed steps (256 MiB write, outside the step events)"}


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled every 50 ms during the timed region,
    through NVML in-process (the library nvidia-smi reads; a process spawned per sample would
    land in the timed region), on the device torch runs on (matched by UUID).  Falls back to
    one `nvidia-smi -lms 200` process when pynvml is missing."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, device: torch.device):
        self.device = device
        self.samples = []  # (sm_mhz, sm_max_mhz, watts, reason bits)
        self._stop = threading.Event()
        self._t = None
        self._nv = None
        self._h = None
        try:
            import pynvml

            pynvml.nvmlInit()
            uuid = str(torch.cuda.get_device_properties(device).uuid)
            for i in range(pynvml.nvmlDeviceGetCount()):
                h = pynvml.nvmlDeviceGetHandleByIndex(i)
                u = pynvml.nvmlDeviceGetUUID(h)
                u = u.decode() if isinstance(u, bytes) else u
                if u.replace("GPU-", "") == uuid.replace("GPU-", ""):
                    self._nv, self._h = pynvml, h
                    break
        except Exception:
            self._nv = None

    def _run(self):
        nv, h = self._nv, self._h
        while not self._stop.is_set():
            try:
                self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                     nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM),
                                     nv.nvmlDeviceGetPowerUsage(h) / 1000.0,
                                     int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))))
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        if os.environ.get("DFSS_BENCH_NO_SAMPLER"):  # (diagnostics: timing without the sampling thread)
            return self
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        else:
            self._p = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, text=True)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)
        elif getattr(self, "_p", None):
            self._p.terminate()
            for line in self._p.communicate(timeout=5)[0].splitlines():
                f = [x.strip() for x in line.split(",")]
                try:
                    self.samples.append((float(f[0]), float(f[1]), float(f[2]), int(f[3], 16)))
                except (ValueError, IndexError):
                    pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        bits = 0
        for smp in self.samples:
            bits |= smp[3]
        return {"sm_mhz": float(np.median([smp[0] for smp in self.samples])),
                "sm_max_mhz": float(max(smp[1] for smp in self.samples)),
                "power_w": round(float(np.median([smp[2] for smp in self.samples])), 1),
                "reasons": sorted(k for k, b in self.REASONS.items() if bits & b),
                "samples": len(self.samples), "source": "nvml" if self._nv is not None else "nvidia-smi -lms 200"}


def soak(fn, seconds: float | None = None):
    """Run fn back to back for `seconds` (DFSS_BENCH_SOAK_S, default 1.5): a 1 kW B200 reaches its
    sustained (power-capped) clock within about a second of full load, and every arm -- DFSS and
    the dense comparators -- is timed in that same state (tools/time_soak.py: both settle at
    the sw_power_cap clock, SDPA lower than DFSS)."""
    seconds = float(os.environ.get("DFSS_BENCH_SOAK_S", "1.5")) if seconds is None else seconds
    t_end = time.perf_counter() + seconds
    while time.perf_counter() < t_end:
        for _ in range(20):
            fn()
        torch.cuda.synchronize()


def soaked_steps(fn, steps, warmup, flush, device):
    """soak, then time_steps, under one clock sampler: (per-step ms, clocks)."""
    with ClockSampler(device) as clk:
        soak(fn)
        times = time_steps(fn, steps, warmup, flush)
    return times, clk.summary()


def time_steps(fn, steps, warmup, flush=None):
    """Per-step CUDA events on the current stream; L2 flushed between steps outside the events."""
    # warm-up steps exactly like the timed ones (flush included): after unflushed warm-up steps
    # the first flushed step of the fused kernel ran ~2x the others (c2 0.107 vs 0.049 ms,
    # tools/time_firststep.py), an artefact of the harness, not a property of the step
    for _ in range(warmup):
        if flush is not None:
            flush()
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for s, e in ev:
        if flush is not None:
            flush()
        s.record()
        fn()
        e.record()
    torch.cuda.synchronize()
    return [s.elapsed_time(e) for s, e in ev]


def kernel_stats(cfg_name: str, key: str) -> dict:
    p = os.path.join(ROOT, "profiles", "ncu_kernel_stats.json")
    try:
        return json.load(open(p)).get(cfg_name, {}).get(key, {}) or {}
    except (OSError, ValueError):
        return {}


#: kernels one dfss_attention call launches on each path (dfss_nm_attention, capi.cu)
LAUNCHES = {"fused-16bit": 1, "fused-tf32": 2, "staged-tcgen05": 2, "staged-ffma": 2, "staged-masked": 3,
            "staged-3xtf32": 4}


def roofline(cfg_name: str, path: str, ms: float, bh: int) -> dict:
    """Binding floor of the kernel(s) of one step, and the measured time against it.

    Fused paths (one kernel): HBM floor = Q, K, V read + O written (4 n d bytes-per-element
    per head); tensor floor = 3 n^2 d flops per head at the dense rate (QK^T 2 n^2 d dense,
    P.V n^2 d dense-equivalent at the 2x sparse rate).  Staged exact-FP32 path: HBM floor = the
    staged bytes (SDDMM writes nonzeros + metadata, the softmax-fused SpMM reads them: 4.5 n^2 +
    16 n d per head for 1:2 fp32, SURVEY §8(d) with the softmax fused) and FFMA floor = 3 n^2 d on
    the FP32 pipe.  `frac` = max(floors) / measured; `bound` names the larger floor; `achieved`
    and `peak` are in that floor's unit.  The issue-rate floor (ncu warp instructions per launch
    / (4 schedulers x SMs x max clock)) is the practical bound of the epilogue-bound fused kernel."""
    cfg = CONFIGS[cfg_name]
    n, d = cfg["seq"], cfg["d"]
    eb = 4 if cfg["dtype"] == "float32" else 2
    hbm, tf_bf16, sm_mhz, src = peaks()
    t = ms * 1e-3
    if path.startswith("fused"):
        nbytes = 4 * n * d * eb * bh
        flops = 3.0 * n * n * d * bh
        tf = tf_bf16 if path == "fused-16bit" else tf_bf16 / 2  # tf32 dense = half the 16-bit rate
        floors = {"hbm": nbytes / (hbm * 1e9), "tensor": flops / (tf * 1e12)}
        kname = ("dfss_flash2_kernel" if n % 256 == 0 else "dfss_flash_kernel") if path == "fused-16bit" \
            else "dfss_flash_tf32_kernel"
        stats = kernel_stats(cfg_name, "flash" if path == "fused-16bit" else "flashtf32")
        peak_tensor = (f"MEASURED_PEAKS.json bf16_tflops ({src})" if path == "fused-16bit" else
                       f"MEASURED_PEAKS.json bf16_tflops / 2 for tf32 ({src})")
    elif path == "staged-3xtf32":
        # scores (3 tf32 passes of QK^T) + row maxima, SpMM with the softmax fused (3 sparse tf32
        # passes); bytes: the nonzeros written and read once, metadata written / read, and Q / K / V
        # read and split into hi / lo, O written
        nz = n * (n // 2) * eb
        meta = n * (n // 2) // 2
        nbytes = (2 * nz + 2 * meta + 16 * n * d * eb) * bh
        flops = 3.0 * 3.0 * n * n * d * bh
        tf = tf_bf16 / 2
        floors = {"hbm": nbytes / (hbm * 1e9), "tensor": flops / (tf * 1e12)}
        kname = "sddmm12_tf32x3_kernel + spmm12_tf32x3_kernel (staged 3xTF32, softmax fused)"
        stats = {}
        peak_tensor = f"MEASURED_PEAKS.json bf16_tflops / 2 for tf32 ({src})"
    else:
        gs = 2 if cfg["mode"] == "1:2" else 4
        nz = n * (n // 2) * eb
        meta = n * (n // gs) // 2
        nbytes = (2 * (nz + meta) + 4 * n * d * eb) * bh
        flops = 3.0 * n * n * d * bh
        tf = FP32_FFMA_TFLOPS
        floors = {"hbm": nbytes / (hbm * 1e9), "fp32_ffma": flops / (tf * 1e12)}
        kname = "sddmm_simt_kernel + spmm_simt_softmax (staged exact FP32)"
        stats = kernel_stats(cfg_name, "spmm")
        peak_tensor = "nominal FP32 FFMA 148 SMs x 128 FMA/clk x 2 x 1.965 GHz (not in MEASURED_PEAKS.json)"
    bound = max(floors, key=floors.get)
    if bound == "hbm":
        achieved, peak, unit, psrc = nbytes / t / 1e9, hbm, "GB/s", f"MEASURED_PEAKS.json hbm_gbs ({src})"
    else:
        achieved, peak, unit, psrc = flops / t / 1e12, tf, "TFLOP/s", peak_tensor
    out = {"kernel": kname, "bound": bound, "achieved": round(achieved, 1), "peak": round(peak, 1), "unit": unit,
           "frac": round(floors[bound] / t, 4), "traffic": stats.get("traffic"), "peak_source": psrc,
           "floors_us": {k: round(v * 1e6, 2) for k, v in floors.items()}, "measured_us": round(t * 1e6, 2),
           "algorithmic_bytes_per_launch": int(nbytes), "algorithmic_flops_per_launch": flops}
    if stats.get("warp_instructions"):
        issue_s = float(stats["warp_instructions"]) / (4 * 148 * sm_mhz * 1e6)
        out["issue_floor_us"] = round(issue_s * 1e6, 2)
        out["issue_frac"] = round(issue_s / t, 4)
        out["ncu_capture"] = stats.get("capture")
    return out


def run_dfss(args, cfg_name, ws, rank, local, device, report_extra=True, info=True, scaling="weak"):
    import paper_2203_00091_b200 as dfss

    cfg = CONFIGS[cfg_name]
    n, d = cfg["seq"], cfg["d"]
    total_bh = job_heads(cfg, ws, scaling)
    lo, hi = shard(total_bh, ws, rank)
    qkv = make_inputs(cfg, lo, hi, device)
    q, k, v = qkv[0], qkv[1], qkv[2]
    bh = hi - lo
    mode = dfss.SparsityMode.parse(cfg["mode"])
    math_mode = cfg.get("math", "auto")
    path = dfss.attention_path(mode, q.dtype, n, d, math_mode, bh=max(bh, 1))
    ws_bytes = dfss.workspace_bytes(mode, q.dtype, max(bh, 1), n, d, math_mode)
    workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=device)
    out = torch.empty_like(q)
    flush_buf = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=device)
    flush = lambda: flush_buf.fill_(1)  # noqa: E731

    def step():
        if bh:
            dfss.dfss_attention(q, k, v, mode, math_mode=math_mode, out=out, workspace=workspace)

    # ---- timed region: barrier + synchronize on both sides, max over ranks
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    # soak (sustained-load clocks, see soak()), then the K timed steps, one sampler window
    times, clocks = soaked_steps(step, args.steps, args.warmup, flush, device)
    if os.environ.get("DFSS_BENCH_STEP_TIMES"):
        print(f"[bench] {cfg_name} step ms: " + " ".join(f"{x:.4f}" for x in times), file=sys.stderr)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    total_ms = torch.tensor([sum(times)], dtype=torch.float64, device=device)
    if ws > 1:
        torch.distributed.all_reduce(total_ms, op=torch.distributed.ReduceOp.MAX)
    ms_per_step = float(total_ms.item()) / args.steps
    value = 4.0 * n * n * d * total_bh / (ms_per_step * 1e-3) / 1e12  # all ranks' heads / max-rank time
    res = {"ms_per_step": ms_per_step, "value": value, "clocks": clocks, "bh_local": bh, "path": path,
           "launches_per_step": LAUNCHES[path] if bh else 0, "lo": lo, "hi": hi}
    if not report_extra:
        return res, (q, k, v, out, lo, hi)
    res["roofline"] = roofline(cfg_name, path, ms_per_step, bh)

    # ---- dense baselines on the same box and shard: unfused cuBLAS (the paper's "full
    # attention", scale folded into Q) and fused SDPA (flash / cuDNN)
    scale = 1.0 / math.sqrt(d)
    qd, kd, vd = q.unsqueeze(0), k.unsqueeze(0), v.unsqueeze(0)

    def dense_unfused():
        s = torch.matmul(q * scale, k.transpose(-1, -2))
        return torch.matmul(torch.softmax(s, dim=-1), v)

    def dense_sdpa():
        return torch.nn.functional.scaled_dot_product_attention(qd, kd, vd)

    base, base_clk = {}, {}
    for name, fn in (("cublas_unfused", dense_unfused), ("sdpa", dense_sdpa)):
        try:  # same protocol as the DFSS step: soaked to the sustained clock, L2 flushed per step
            tt, base_clk[name] = soaked_steps(fn, max(3, args.steps), 2, flush, device)
            base[name] = float(np.mean(tt))
        except Exception as ex:  # e.g. OOM for huge unfused scores
            base[name] = None
            res.setdefault("baseline_errors", {})[name] = str(ex)[:120]
    res["dense_ms"] = base
    res["dense_clocks"] = base_clk
    res["speedup_vs_dense"] = {k_: (round(t / ms_per_step, 3) if t else None) for k_, t in base.items()}

    # ---- staged reference-shaped kernels on the same shard (informational: sddmm_prune ->
    # softmax_rows -> spmm, the three-kernel path the paper describes)
    if info and path == "fused-16bit" and cfg["mode"] == "2:4":
        holder = {}

        def k_sddmm():
            holder["c"], _ = dfss.sddmm_prune(q, k, mode, scale, with_row_max=True)

        def k_spmm_softmax():
            dfss.spmm_softmax(holder["c"], v)

        k_sddmm()
        res["staged_kernels_ms"] = {
            "sddmm_rowmax": float(np.mean(time_steps(k_sddmm, max(3, args.steps), 2, flush))),
            "spmm_softmax": float(np.mean(time_steps(k_spmm_softmax, max(3, args.steps), 2, flush)))}
    del workspace, flush_buf
    return res, (q, k, v, out, lo, hi)


def parity_spot_check(cfg_name, q, k, v, out, lo, hi, total_bh):
    """Oracle check of heads from the first, middle and last persistent-CTA rounds of the timed
    output (the two first, one middle and the two last heads of this shard); SURVEY §8(c)
    tolerances: 1e-5 for exact FP32, 2e-2 for 16-bit and tf32 (on tf32-truncated operands)."""
    from oracle import oracle_c

    cfg = CONFIGS[cfg_name]
    bh = hi - lo
    if bh == 0:
        return {"heads": [], "ok": True}
    idx = sorted({0, min(1, bh - 1), bh // 2, max(bh - 2, 0), bh - 1})
    x = [t[idx].double().cpu().numpy() for t in (q, k, v)]
    if cfg.get("math") == "tf32":
        x = [(a.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32).astype(np.float64)
             for a in x]
    want = oracle_c.attention_batched(x[0], x[1], x[2], cfg["mode"], nthreads=min(8, len(idx)))
    got = out[idx].double().cpu().numpy()
    tol = 1e-5 if cfg["dtype"] == "float32" and cfg.get("math") != "tf32" else 2e-2
    err = np.abs(got - want)
    ok = bool((err <= tol + tol * np.abs(want)).all())
    return {"heads": [lo + i for i in idx], "of": total_bh, "tol": tol, "ok": ok, "max_abs_err": float(err.max())}


def e2e_measure(args, cfg, q, k, v, device, ws, total_bh):
    """Same metric through the public host-buffer API (dfss_attention_host, synchronous like the
    reference's calls) with pinned host buffers: every step copies Q/K/V host->device, runs the
    kernel and copies O back, pipelined over 4 batch x heads pieces on three streams.  Max over
    ranks when N > 1."""
    import paper_2203_00091_b200 as dfss

    mode = dfss.SparsityMode.parse(cfg["mode"])
    hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
    hout = torch.empty(q.shape, dtype=q.dtype).pin_memory()
    math_mode = cfg.get("math", "auto")

    def step():
        if q.shape[0]:
            dfss.dfss_attention_host(hq, hk, hv, mode, math_mode=math_mode, out=hout, chunks=4, device=device)

    if ws > 1:
        torch.distributed.barrier()
    ms = float(np.mean(time_steps(step, max(3, args.steps), 2)))
    if ws > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    n, d = cfg["seq"], cfg["d"]
    eb = q.element_size()
    return {"ms_per_step": ms, "value": 4.0 * n * n * d * total_bh / (ms * 1e-3) / 1e12, "unit": UNIT,
            "h2d_bytes_per_step": 3 * int(q.shape[0]) * n * d * eb, "d2h_bytes_per_step": int(q.shape[0]) * n * d * eb,
            "api": "dfss_attention_host (pinned host tensors in and out, synchronous)"}


def cpu_reference(cfg, budget_s: float, threads: int, dense: bool = False):
    """The reference's CPU algorithm (C restatement of nmattn.nm_attention, or of full_attention
    with dense=True; float64, the numba kernels' operation order) on a bounded sample of the
    workload's heads, all host threads."""
    from oracle import oracle_c

    n, d = cfg["seq"], cfg["d"]
    total_bh = cfg["batch"] * cfg["heads"]
    qkv = make_inputs(cfg, 0, 1, "cpu")
    x = [t.double().numpy() for t in qkv]
    t0 = time.perf_counter()
    oracle_c.attention_batched(x[0], x[1], x[2], cfg["mode"], nthreads=1, dense=dense)
    per_head = time.perf_counter() - t0
    heads = int(max(threads, min(total_bh, budget_s * threads / max(per_head, 1e-6))))
    heads = max(1, min(total_bh, heads - heads % threads if heads >= threads else heads))
    qkv = make_inputs(cfg, 0, heads, "cpu")
    x = [t.double().numpy() for t in qkv]
    t0 = time.perf_counter()
    oracle_c.attention_batched(x[0], x[1], x[2], cfg["mode"], nthreads=threads, dense=dense)
    el = time.perf_counter() - t0
    what = "full_attention (dense fp64)" if dense else "nm_attention"
    return {"value": 4.0 * n * n * d * heads / el / 1e12, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{heads} of {total_bh} (batch x head) slices, float64 C restatement of nmattn.{what} "
                      f"(oracle/dfss_oracle.c, bitwise the numba reference on tests/golden), {el:.2f} s wall, "
                      f"{per_head * 1e3:.1f} ms/head single-core",
            "seconds": el, "heads": heads, "ms_per_head_1core": per_head * 1e3}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def block_mask_measure(device, steps=5):
    """BlockMask tile skipping on the c4 shape (batch 8, 12 heads, seq 4096,
    2:4 bf16).  Block-causal mask at 128 x 128 granularity on (32, 64) tiles: fully masked steps
    are skipped (no K / V load, MMA or softmax work).  Dense SDPA with is_causal=True is listed as
    the closest dense counterpart (token-causal, not block-causal)."""
    import paper_2203_00091_b200 as dfss

    b, h, n, d = 8, 12, 4096, 64
    g = torch.Generator(device="cpu").manual_seed(5)
    q, k, v = (torch.randn((b, h, n, d), generator=g).to(torch.bfloat16).to(device) for _ in range(3))
    out = torch.empty_like(q)
    rows, cols = np.arange(n // 32) * 32 // 128, np.arange(n // 64) * 64 // 128
    keep = cols[None, :] <= rows[:, None]
    mask = dfss.BlockMask(keep, 32, 64)
    ws = torch.empty(dfss.workspace_bytes("2:4", q.dtype, b * h, n, d, block_mask=mask), dtype=torch.uint8,
                     device=device)
    flush_buf = torch.empty(256 * 2**20, dtype=torch.uint8, device=device)
    flush = lambda: flush_buf.fill_(1)  # noqa: E731
    t = lambda fn: float(np.mean(soaked_steps(fn, steps, 3, flush, device)[0]))  # noqa: E731
    res = {"workload": "c4 shape, 2:4 bf16, block-causal 128x128 BlockMask on 32x64 tiles",
           "live_step_fraction": round(float(keep[::4, ::2].mean()), 4),
           "dfss_unmasked_ms": round(t(lambda: dfss.dfss_attention(q, k, v, "2:4", out=out)), 4),
           "dfss_block_causal_ms": round(t(lambda: dfss.dfss_attention(q, k, v, "2:4", block_mask=mask, out=out,
                                                                        workspace=ws)), 4)}
    sdpa = torch.nn.functional.scaled_dot_product_attention
    res["sdpa_dense_ms"] = round(t(lambda: sdpa(q, k, v)), 4)
    res["sdpa_causal_ms"] = round(t(lambda: sdpa(q, k, v, is_causal=True)), 4)
    res["speedup_vs_unmasked"] = round(res["dfss_unmasked_ms"] / res["dfss_block_causal_ms"], 3)
    res["speedup_vs_sdpa_causal"] = round(res["sdpa_causal_ms"] / res["dfss_block_causal_ms"], 3)
    return res


def reference_arm(args, ws, rank, threads):
    """--impl reference: the reference's CPU algorithm on the host cores, rank 0 only."""
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    steps = []
    budget = max(2.0, min(20.0, 150.0 / (args.steps + args.warmup)))
    for i in range(args.warmup + args.steps):
        r = cpu_reference(cfg, budget, threads)
        if i >= args.warmup:
            steps.append(r)
    dense = cpu_reference(cfg, min(budget, 10.0), threads, dense=True)
    val = float(np.median([s["value"] for s in steps]))
    secs = float(np.median([s["seconds"] for s in steps]))
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1e3, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(args.config, args.gpus, args.scaling, steps[-1]["heads"]),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": steps[-1]["sample"], "cpu_model": cpu_model()},
            "cpu_full_attention": {"value": dense["value"], "unit": UNIT, "cores": threads, "sample": dense["sample"]},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["dfss", "reference"], default="dfss")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--no-sweep", action="store_true", help="skip the configs[4] sequence sweep")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of CPU work for the CPU baseline")
    ap.add_argument("--no-extra", action="store_true", help="skip sweep / e2e / cpu baseline (profiling runs)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    ws, rank, local = dist_env()
    cfg = CONFIGS[args.config]
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    if args.impl == "reference":
        return reference_arm(args, ws, rank, threads)

    if ws > 1:
        torch.cuda.set_device(local)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    device = torch.device("cuda", torch.cuda.current_device())

    res, (q, k, v, out, lo, hi) = run_dfss(args, args.config, ws, rank, local, device, scaling=args.scaling)
    total_bh = job_heads(cfg, ws, args.scaling)

    # end-to-end parity gather: NCCL all_gather of the output shards (outside the timed region);
    # shards are padded to the largest one (strong scaling may split unevenly)
    parity = None
    if ws > 1:
        width = max(b - a for a, b in (shard(total_bh, ws, r) for r in range(ws)))
        pad = torch.zeros((width,) + tuple(out.shape[1:]), dtype=out.dtype, device=device)
        pad[: hi - lo] = out
        gathered = torch.empty((width * ws,) + tuple(out.shape[1:]), dtype=out.dtype, device=device)
        torch.distributed.all_gather_into_tensor(gathered, pad)
        parts = [gathered[r * width: r * width + (shard(total_bh, ws, r)[1] - shard(total_bh, ws, r)[0])]
                 for r in range(ws)]
        full = torch.cat(parts)
        parity = {"gathered_heads": int(full.shape[0]), "checksum": float(full.float().abs().sum()),
                  "shards_equal_local": bool(torch.equal(full[lo:hi], out))}

    extra = {}
    if not args.no_extra:
        extra["e2e"] = e2e_measure(args, cfg, q, k, v, device, ws, total_bh)
    if rank == 0 and not args.no_extra:
        extra["parity_spot_check"] = parity_spot_check(args.config, q, k, v, out, lo, hi, total_bh)
        budget = args.cpu_budget if ws == 1 else min(args.cpu_budget, 8.0)
        cb = cpu_reference(cfg, budget, threads)
        cb["cpu_model"] = cpu_model()
        extra["cpu_baseline"] = cb
        cd = cpu_reference(cfg, min(budget, 8.0), threads, dense=True)
        extra["cpu_full_attention"] = {"value": cd["value"], "unit": UNIT, "cores": threads, "sample": cd["sample"]}
        if ws == 1:
            others = {}
            for name in ("c1", "c2", "c3", "c4"):
                if name == args.config:
                    continue
                try:
                    r2, (q2, k2, v2, o2, lo2, hi2) = run_dfss(argparse.Namespace(steps=max(3, args.steps // 2),
                                                                                 warmup=3), name, 1, 0, 0, device)
                    others[name] = {"ms_per_step": round(r2["ms_per_step"], 4), "tflops": round(r2["value"], 2),
                                    "speedup_vs_dense": r2["speedup_vs_dense"], "dense_ms": r2["dense_ms"],
                                    "clocks": r2["clocks"], "dense_clocks": r2.get("dense_clocks"),
                                    "path": r2["path"], "gpu_launches_per_step": r2["launches_per_step"],
                                    "roofline": r2["roofline"],
                                    "parity_spot_check": parity_spot_check(name, q2, k2, v2, o2, lo2, hi2, hi2 - lo2)}
                    if "staged_kernels_ms" in r2:
                        others[name]["staged_kernels_ms"] = r2["staged_kernels_ms"]
                    del q2, k2, v2, o2
                except Exception as ex:
                    others[name] = {"error": str(ex)[:200]}
            extra["other_configs"] = others
            if not args.no_sweep:
                sw = {}
                for name in sorted((c for c in CONFIGS if c.startswith("c5_")),
                                   key=lambda c: (c.split("_")[1], int(c.split("_")[2]))):
                    try:
                        r2, _ = run_dfss(argparse.Namespace(steps=5, warmup=3), name, 1, 0, 0, device, info=False)
                        sw[name] = {"ms": round(r2["ms_per_step"], 4), "tflops": round(r2["value"], 1),
                                    "speedup_vs_dense": r2["speedup_vs_dense"], "path": r2["path"],
                                    "frac": r2["roofline"]["frac"], "bound": r2["roofline"]["bound"]}
                    except Exception as ex:
                        sw[name] = {"error": str(ex)[:200]}
                extra["sweep"] = sw
                try:
                    extra["block_mask"] = block_mask_measure(device)
                except Exception as ex:
                    extra["block_mask"] = {"error": str(ex)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(res["value"], 3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(res["ms_per_step"], 5), "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": DTYPE_TAG[cfg["dtype"]],
            "data": "synthetic N(0,1) Q/K/V, seeded per (seed, global head)",
            "config": config_block(args.config, ws, args.scaling, res["bh_local"]),
            "roofline": res["roofline"], "path": res["path"],
            "dense_ms": res["dense_ms"], "speedup_vs_dense": res["speedup_vs_dense"],
            "gpu_launches": res["launches_per_step"] * args.steps, "clocks": res["clocks"],
            "dense_clocks": res.get("dense_clocks"),
        }
        if "staged_kernels_ms" in res:
            line["staged_kernels_ms"] = res["staged_kernels_ms"]
        if "e2e" in extra:
            e = extra.pop("e2e")
            line["e2e"] = {"value": round(e["value"], 3), "unit": e["unit"], "h2d_bytes_per_step": e["h2d_bytes_per_step"],
                           "d2h_bytes_per_step": e["d2h_bytes_per_step"], "ms_per_step": round(e["ms_per_step"], 4),
                           "api": e["api"]}
        if "cpu_baseline" in extra:
            line["cpu_baseline"] = extra.pop("cpu_baseline")
        if parity:
            line["allgather_check"] = parity
        line.update(extra)
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
