"""Calibrates the CPU baseline (run in the build container, where /root/reference exists): the
reference's own nm_attention (numba backend, single-threaded) against the C restatement the
bench's reference arm runs (oracle/dfss_oracle.c, 1 thread), same inputs -- speed per head and
the largest output difference.  Output: profiles/cpu_baseline_calibration.txt."""
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import nmattn  # noqa: E402
from nmattn import backend  # noqa: E402

from oracle import oracle_c  # noqa: E402

rng = np.random.default_rng(0)
lines = [f"reference backend: {backend.active_backend()}"]
for mode in ("2:4", "1:2"):
    for n in (384, 512, 1024):
        q, k, v = (rng.standard_normal((n, 64)) for _ in range(3))
        inp = nmattn.AttentionInputs(nmattn.DenseMatrix(q), nmattn.DenseMatrix(k), nmattn.DenseMatrix(v))
        m = nmattn.SparsityMode.parse(mode)
        ref = np.asarray(nmattn.nm_attention(inp, m).data)  # jit warm-up + result
        reps = 3
        t0 = time.perf_counter()
        for _ in range(reps):
            nmattn.nm_attention(inp, m)
        tn = (time.perf_counter() - t0) / reps
        t0 = time.perf_counter()
        for _ in range(reps):
            port = oracle_c.attention_batched(q[None], k[None], v[None], mode, nthreads=1)[0]
        tc = (time.perf_counter() - t0) / reps
        lines.append(f"{mode} n={n}: reference nm_attention (numba) {tn * 1e3:.1f} ms/head, C port {tc * 1e3:.1f} "
                     f"ms/head, port/reference time {tc / tn:.2f}, max |diff| {np.abs(ref - port).max():.1e}")
out = "\n".join(lines)
print(out)
open(__file__.rsplit("/tools/", 1)[0] + "/profiles/cpu_baseline_calibration.txt", "w").write(out + "\n")
