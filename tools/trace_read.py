import sys, numpy as np
tr = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(16, 2, 64, 2).astype(np.int64)
base = tr[tr > 0].min()
names = {0: "sm s_full ok", 1: "sm computed", 2: "sm p_full arr", 3: "S wait free", 4: "S free ok", 5: "S committed",
         6: "PV p_full ok", 7: "PV committed", 8: "K tma issued", 9: "V tma issued", 10: "S k_full ok"}
it = int(sys.argv[2]) if len(sys.argv) > 2 else 1
for t in range(int(sys.argv[3]) if len(sys.argv) > 3 else 12):
    for h in range(2):
        row = [f"{names[s][:12]}={(tr[s, it, t, h] - base) if tr[s, it, t, h] else -1:7d}" for s in (8, 9, 10, 3, 4, 5, 0, 1, 2, 6, 7) if not (s in (8, 9, 10) and h == 1)]
        print(f"t={t:2d} h={h} " + " ".join(row))
# steady-state deltas (item 1, tiles 8..56)
d = lambda a, b: np.median([tr[b, it, t, h] - tr[a, it, t, h] for t in range(8, 56) for h in range(2)])
print("median per-step:", "s_full->computed", d(0, 1), "computed->p_full", d(1, 2), "p_full(arr)->PV ok", d(2, 6),
      "S free ok -> committed", d(4, 5))
per_tile = np.median(np.diff(tr[0, it, 8:56, 0]))
print("median tile period (set 0):", per_tile)
print("S committed -> sm s_full ok (same tile):", np.median([tr[0, it, t, h] - tr[5, it, t, h] for t in range(8, 56) for h in range(2)]))
print("sm p_full arrive(t) -> S free ok (t+3):", np.median([tr[4, it, t + 3, h] - tr[2, it, t, h] for t in range(8, 56) for h in range(2)]))
