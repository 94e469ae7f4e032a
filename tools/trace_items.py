"""CTA-0 event timeline of the first two items of the two-set kernel (trace build, bring-up):
per step (t, h) the clock of each pipeline event relative to the CTA start, and the per-CTA unit
table, for a small-n config where per-item costs dominate (default c2 = 32,12,512,64).

    bash tools/exp_build.sh trace "-DDFSS_FLASH_TRACE_BUILD"
    DFSS_LIB=exp/trace/libdfss_sm100a.so python tools/trace_items.py gpurun_out/items.bin
"""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
out_file = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/items.bin"
NAMES = {0: "s_full ok", 11: "ld ch0", 12: "cmp ch0", 13: "ld ch1", 14: "cmp ch1", 1: "computed", 2: "p_full arr",
         3: "S wait free", 4: "S free ok", 5: "S commit", 10: "S k_full ok", 6: "PV start", 7: "PV commit",
         8: "K issue", 9: "V issue"}
if os.environ.get("DFSS_FLASH_TRACE") is None:
    subprocess.run([sys.executable, __file__, out_file], env=dict(os.environ, DFSS_FLASH_TRACE=out_file), check=True)
    raw = np.fromfile(out_file, dtype=np.uint64).astype(np.int64)
    tr = raw[: 16 * 2 * 64 * 2].reshape(16, 2, 64, 2)
    u = raw[16 * 2 * 64 * 2:].reshape(148, 16, 8)
    t0 = tr[15, 0, 0, 0]
    T = int(os.environ.get("TRACE_T", "4"))
    print("CTA 0: setup done at", tr[15, 0, 1, 0] - t0)
    for it in range(2):
        for t in range(T):
            for h in range(2):
                ev = {NAMES[s]: tr[s, it, t, h] - t0 for s in NAMES if tr[s, it, t, h] > 0}
                print(f"item {it} t {t} h {h}: " + "  ".join(f"{k} {v}" for k, v in sorted(ev.items(), key=lambda x: x[1])))
    base = u[0, 0, 0]
    for b in (0, 1, 147):
        for k in range(1, 6):
            e = u[b, k]
            if e[5] > 0:
                print(f"cta {b} unit {k} epilogue: o_full wait {e[4] - e[5]}  LDTM O {e[6] - e[4]}  normalise+store {e[7] - e[6]}"
                      f"  | previous item's O_0 complete (PV issuer) at {u[b, k - 1, 1] - e[5]} rel. to epilogue start")
    for b in (0, 1, 147):
        print(f"cta {b}: " + " | ".join(f"u{k} {[int(x - base) if x > 0 else -1 for x in u[b, k, :8]]}" for k in range(7)))
    sys.exit(0)
import torch  # noqa: E402

import paper_2203_00091_b200 as dfss  # noqa: E402

shape = [int(x) for x in os.environ.get("TRACE_SHAPE", "32,12,512,64").split(",")]
q, k, v = (torch.randn(*shape, device="cuda", dtype=torch.bfloat16) for _ in range(3))
for _ in range(3):
    dfss.dfss_attention(q, k, v, "2:4")
torch.cuda.synchronize()
