"""Diagnostic: round-0 client shifts l_i and D_i of the engine vs the CPU oracle (x0 = 0)."""
import os, sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2410_08760_b200 import data as D
from paper_2410_08760_b200.engine import FedNLEngine
from oracle import fednl_oracle as O
name = sys.argv[1]
shards = D.baseline_shards(name)
cfg = D.baseline_run_config(name, rounds=3)
d = shards[0].dim; lam = shards[0].lam
eng = FedNLEngine(cfg, d, len(shards), shards[0].n_samples, lam=lam)
eng.upload([s.bmat for s in shards]); eng.init_state()
eng.run_rounds(1)
sc, cs = eng.round_scalars()
w = d * (d + 1) // 2
diag_idx = np.array([j * (j + 1) // 2 + j for j in range(d)])
wt = np.full(w, 2.0); wt[diag_idx] = 1.0
bad = 0
for c in range(len(shards)):
    ev = O.local_eval(shards[c].bmat, lam, np.zeros(d), need_hess=True, need_f=False)
    Dv = ev.hess.copy(); Dv[diag_idx] -= lam
    l = np.sqrt(np.sum(wt * Dv * Dv))
    dd = eng.round_diff(c)
    ld = np.sqrt(np.sum(wt * dd * dd))
    if abs(l - cs[c]) > 1e-10 * l:
        bad += 1
        if bad < 4: print(c, cs[c], l, ld, np.abs(dd - Dv).max())
print(name, "bad", bad)
