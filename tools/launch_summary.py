"""Mean per-kernel duration from ncu --metrics gpu__time_duration.sum CSV launch lists.

    python tools/launch_summary.py gpurun_out/launches_*.csv
"""
import collections
import csv
import sys

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    if not rows:
        continue
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = collections.defaultdict(list)
    for r in rows[1:]:
        d[r[ki][:80]].append(float(r[vi].replace(",", "")))
    print(f)
    for k, v in d.items():
        print(f"  {len(v):4d} {sum(v) / len(v) / 1000:10.1f} us  {k}")
