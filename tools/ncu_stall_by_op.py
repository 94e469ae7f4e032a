"""Stall reasons per SASS opcode from an ncu --set full capture (bring-up tool).

    python tools/ncu_stall_by_op.py <report.ncu-rep> [min_samples]

Rows: opcode classes; columns: the main per-warp stall reasons (samples), so the waits
(long scoreboard on LDTM / try_wait, math-pipe throttle on the ALU, dispatch) can be attributed.
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO("\n".join(out.splitlines()[1:]))))
h = rows[0]
cols = ["stall_long_sb", "stall_math", "stall_dispatch", "stall_wait", "stall_short_sb", "stall_barrier",
        "stall_not_selected", "stall_selected", "stall_branch_resolving", "stall_no_inst", "stall_sleep"]
ci = [h.index(c) for c in cols]
isrc = h.index("Source")
agg = collections.defaultdict(lambda: [0] * len(cols))
for r in rows[1:]:
    try:
        vals = [int(r[i]) for i in ci]
    except (ValueError, IndexError):
        continue
    s = r[isrc].strip()
    op = s.split()[1] if s.startswith("@") else s.split()[0]
    op = op.split(".")[0]
    for j, v in enumerate(vals):
        agg[op][j] += v
tot = [sum(a[j] for a in agg.values()) for j in range(len(cols))]
print("op          " + " ".join(f"{c[6:14]:>9s}" for c in cols))
print("TOTAL       " + " ".join(f"{t:9d}" for t in tot))
for op, a in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:25]:
    print(f"{op:12s}" + " ".join(f"{v:9d}" for v in a))
