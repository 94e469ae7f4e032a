import sys, numpy as np
tr = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(16, 2, 64, 2).astype(np.int64)
T = int(sys.argv[2]) if len(sys.argv) > 2 else 32
it = 1
rng = range(4, T - 4)
d = lambda a, b, off=0: np.median([tr[b, it, t + off, h] - tr[a, it, t, h] for t in rng for h in range(2)])
print(f"{sys.argv[1]}: period set0 {np.median(np.diff(tr[0, it, 4:T-4, 0])):.0f} | compute {d(0, 1):.0f} | "
      f"p_full->PV ok {d(2, 6):.0f} | PV ok->committed {d(6, 7):.0f} | S free ok->committed {d(4, 5):.0f} | "
      f"S wait free->ok {d(3, 4):.0f} | p_full(t)->s_full(t+1) {d(2, 0, 1):.0f}")
