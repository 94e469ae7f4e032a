"""Summarise ncu captures from gpurun_out/ into profiles/ (run in the build container).

    python tools/ncu_summary.py <tag>

Reads gpurun_out/launches_<tag>_<cfg>.csv (gpu__time_duration launch lists) and
gpurun_out/prof_<tag>_<cfg>_<kernel>.ncu-rep (--set full), writes
profiles/<tag>_ncu_summary.md, copies the launch lists to profiles/, and
updates profiles/ncu_kernel_stats.json (dram bytes and issued warp instructions per launch,
read by bench.py for the roofline traffic and the issue-rate floor).
"""

from __future__ import annotations

import csv
import glob
import io
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "regs",
    "smsp__inst_executed.sum": "warp_insts",
    "smsp__inst_issued.sum": "warp_issued",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6,
              "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "s": 1.0, "nsecond": 1e-9,
              "hz": 1.0, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}


def raw_metrics(rep: str) -> dict:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return {}
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
    for m, key in METRICS.items():
        if m in hdr:
            i = hdr.index(m)
            try:
                v = float(vals[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i].strip()
            if u in UNIT_SCALE:
                v *= UNIT_SCALE[u]
            out[key] = v
    return out


def launch_list(path: str):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    return [(re.sub(r"\(.*", "", r[ki]).replace("void ", ""), float(r[vi].replace(",", "")) * 1e-3)
            for r in data if r[mi] == "gpu__time_duration.sum"]


def main(tag: str) -> None:
    os.makedirs(PROF, exist_ok=True)
    lines = [f"# ncu summary `{tag}`", "",
             "Captured with `tools/profile.sh` / `tools/prof_one.sh` under gpurun on one B200 "
             "(`--clock-control none`; launch lists are cold-cache and serialised, compare shares).", ""]
    traffic_path = os.path.join(PROF, "ncu_kernel_stats.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for path in sorted(glob.glob(os.path.join(OUT, f"launches_{tag}_*.csv"))):
        cfg = path.rsplit("_", 1)[1].replace(".csv", "")
        shutil.copy(path, os.path.join(PROF, os.path.basename(path)))
        seq = [s for s in launch_list(path) if "dfss" in s[0]]
        tot = {}
        for name, us in seq:
            tot.setdefault(name, []).append(us)
        step = sum(sum(v) / len(v) for v in tot.values())
        lines += [f"## launch list {cfg} (`{os.path.basename(path)}`)", "",
                  "| kernel | launches | mean µs | share of DFSS step |", "|---|---|---|---|"]
        for name, v in tot.items():
            m = sum(v) / len(v)
            lines.append(f"| `{name}` | {len(v)} | {m:.1f} | {m / step:.1%} |")
        lines.append("")
    for rep in sorted(glob.glob(os.path.join(OUT, f"prof_{tag}_*.ncu-rep"))):
        base = os.path.basename(rep).replace(".ncu-rep", "")
        cfg = base.split("_")[2]
        m = raw_metrics(rep)
        if not m:
            continue
        kname = re.sub(r"\(.*", "", m["kernel"]).replace("void ", "")
        dram = m.get("dram_read", 0) + m.get("dram_write", 0)
        suffix = base.split("_")[-1]
        key = (suffix if suffix.startswith("flash") and suffix != "flash" else "flash" if "flash" in kname
               else "sddmm" if "sddmm" in kname else "softmax" if "softmax" in kname else "spmm")
        traffic.setdefault(cfg, {})[key] = {"traffic": int(dram), "capture": tag,
                                            "warp_instructions": m.get("warp_issued", m.get("warp_insts", 0))}
        lines += [f"## `{kname}` — {cfg} (`{base}.ncu-rep`)", "",
                  f"- duration {m.get('duration', 0) * 1e6:.1f} µs at SM clock {m.get('sm_clock', 0) / 1e9:.2f} GHz",
                  f"- DRAM traffic {dram / 1e9:.3f} GB (read {m.get('dram_read', 0) / 1e9:.3f}, "
                  f"write {m.get('dram_write', 0) / 1e9:.3f}) = {dram / max(m.get('duration', 1), 1e-12) / 1e9:.0f} GB/s; "
                  f"dram throughput {m.get('dram_pct', 0):.1f}% of peak",
                  f"- tensor pipe {m.get('tensor_pct', 0):.1f}%, ALU pipe {m.get('alu_pct', 0):.1f}%, "
                  f"FMA pipe {m.get('fma_pct', 0):.1f}%, issue active {m.get('issue_pct', 0):.1f}%, "
                  f"warps active {m.get('warps_active_pct', 0):.1f}%, {int(m.get('regs', 0))} regs/thread, "
                  f"{m.get('warp_insts', 0) / 1e6:.1f} M warp-instructions", ""]
    with open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
