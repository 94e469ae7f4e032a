"""Quick read of one ncu report: key SOL / pipe / stall metrics and a SASS opcode histogram.
    python tools/ncu_quick.py gpurun_out/prof_x.ncu-rep [--lines N]"""
import csv, io, subprocess, sys, collections

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]
want = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]
for w in want:
    if w in h:
        i = h.index(w)
        print(f"{w:70s} {u[i]:10s} {v[i]}")
stalls = [(name, float(v[i])) for i, name in enumerate(h) if name.startswith("smsp__average_warp_latency_issue_stalled_") or
          (name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("_not_issued"))]
stalls = [s for s in stalls if s[1] > 0]
for name, val in sorted(stalls, key=lambda x: -x[1])[:14]:
    print(f"  {name:80s} {val}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
iS, iE, iW = hh.index("Source"), hh.index("Instructions Executed"), hh.index("Warp Stall Sampling (All Samples)")
tot, st = collections.Counter(), collections.Counter()
for row in rows[2:]:
    try:
        e, w = int(row[iE]), int(row[iW])
    except (ValueError, IndexError):
        continue
    t = row[iS].strip().split()
    if not t:
        continue
    o = t[1] if t[0].startswith("@") else t[0]
    o = o.rstrip(";")
    tot[o] += e
    st[o] += w
allE = sum(tot.values()); allW = sum(st.values())
print("executed", allE, "stall samples", allW)
for k, val in tot.most_common(28):
    print(f"  {k:32s} {val:12d} {100*val/allE:5.1f}%  stall {100*st[k]/max(allW,1):5.1f}%")
if "--lines" in sys.argv:
    n = int(sys.argv[sys.argv.index("--lines") + 1])
    top = sorted(((int(row[iW]) if row[iW].isdigit() else 0, idx, row[iS].strip()) for idx, row in enumerate(rows[2:])), reverse=True)[:n]
    for w, idx, s in top:
        print(f"  line {idx:5d} stall {w:6d}  {s[:90]}")

if "--reason" in sys.argv:
    col = sys.argv[sys.argv.index("--reason") + 1]
    ic = hh.index(col)
    top = sorted(((int(row[ic]) if row[ic].isdigit() else 0, idx, row[iS].strip()) for idx, row in enumerate(rows[2:])), reverse=True)[:15]
    print("top lines for", col)
    for w, idx, s in top:
        print(f"  line {idx:5d} {w:6d}  {s[:90]}")
