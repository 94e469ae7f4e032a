"""Per-SASS-instruction execution counts and stall samples from an ncu --set full capture.

    python tools/ncu_sass_hot.py <report.ncu-rep> [top]

Prints the instructions with the most executions (and stall samples), plus totals grouped by
opcode, so instruction overhead outside the prune / exp core shows up (bring-up tool).
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
ia, isrc, iex, ismp = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index(
    "Warp Stall Sampling (All Samples)")
ins = []
for r in rows[1:]:
    try:
        ins.append((int(r[ia], 16), r[isrc].strip(), int(r[iex]), int(r[ismp])))
    except (ValueError, IndexError):
        pass
tot = sum(x[2] for x in ins)
smp = sum(x[3] for x in ins)
print(f"total warp instructions {tot}, stall samples {smp}")
byop = collections.Counter()
smop = collections.Counter()
for a, s, e, m in ins:
    op = s.split()[0] if not s.startswith("@") else s.split()[1]
    byop[op.split(".")[0]] += e
    smop[op.split(".")[0]] += m
print("by opcode (executions, % of total, stall samples %):")
for k, v in byop.most_common(40):
    print(f"  {k:12s} {v:12d} {100 * v / tot:6.2f}%  {100 * smop[k] / max(smp, 1):6.2f}%")
# contiguous regions by execution count level
print("hot instructions by stall samples:")
for a, s, e, m in sorted(ins, key=lambda x: -x[3])[:top]:
    print(f"  {a & 0xfffff:06x} {e:10d} {m:7d}  {s[:90]}")

# instructions grouped by execution count (e.g. once per softmax warp-step, per role-warp step)
print("execution-count classes (count: #instructions, total executions):")
cls = collections.defaultdict(lambda: [0, 0])
for a, s, e, m in ins:
    cls[e][0] += 1
    cls[e][1] += e
for e, (n, t) in sorted(cls.items(), key=lambda kv: -kv[1][1])[:15]:
    print(f"  {e:10d} x {n:5d} instr = {t:12d} ({100 * t / tot:5.2f}%)")
