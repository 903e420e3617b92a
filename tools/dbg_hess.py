import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import fednl_oracle as O
from paper_2410_08760_b200 import data as D
from paper_2410_08760_b200.engine import FedNLEngine
d = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
ni = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
shards = D.gaussian_shards(d, n, ni, 1e-4, seed=1)
cfg = D.baseline_run_config("c4", rounds=1)
x = np.zeros(d)
with FedNLEngine(cfg, d, n, ni) as eng:
    eng.upload([s.bmat for s in shards], [s.lam for s in shards])
    f, g, h = eng.oracle_eval(x)
iu = O.tri(d) if hasattr(O, "tri") else None
for c in range(n):
    ev = O.local_eval(shards[c].bmat, shards[c].lam, x)
    diff = np.abs(h[c] - ev.hess)
    bad = np.flatnonzero(diff > 1e-10 * np.max(np.abs(ev.hess)))
    if bad.size:
        # packed t -> (i, j)
        j = np.floor((np.sqrt(8 * bad + 1) - 1) / 2).astype(int)
        i = bad - j * (j + 1) // 2
        tiles = sorted(set(zip((i // 64).tolist(), (j // 64).tolist())))
        cols = sorted(set((j % 64).tolist()))
        print(f"client {c}: {bad.size} bad entries, tiles {tiles[:20]}..({len(tiles)}), tile-cols {cols[:20]}, sample got {h[c][bad[:3]]} want {ev.hess[bad[:3]]}")
    else:
        print(f"client {c}: ok")
