import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import fednl_oracle as O
from paper_2410_08760_b200 import data as D
from paper_2410_08760_b200.engine import FedNLEngine
shards = D.baseline_shards("c0")
cfg = D.baseline_run_config("c0", rounds=4)
d, n = shards[0].dim, len(shards)
run = O.OracleRun(O.OracleConfig.from_run_config(cfg), [s.bmat for s in shards], lam=shards[0].lam, workers=16)
run.init()
for r in range(2): run.fednl_round(r)
x0, hc, hm = run.x.copy(), run.h_cli.copy(), run.h_mas.copy()
gsum = np.zeros(d); shifts = []
for c in range(n):
    ev = O.local_eval(shards[c].bmat, shards[c].lam, x0)
    gsum += ev.grad; shifts.append(O.frob(ev.hess - hc[c], d))
gbar = gsum / n; shift = sum(shifts) / n
p_ref = O.shifted_solve(hm, d, shift, gbar)
eng = FedNLEngine(cfg, d, n, shards[0].n_samples, lam=shards[0].lam)
eng.upload([s.bmat for s in shards]); eng.init_state()
for trial in range(3):
    z = eng.shifted_solve(hm, shift, gbar)
    print("leaf solve rel err", np.max(np.abs(z - p_ref)) / np.max(np.abs(p_ref)))
for trial in range(3):
    eng.set_x(x0); eng.set_client_hest(hc); eng.set_master_hest(hm)
    eng.run_rounds(1, first_round=2)
    sc, cs = eng.round_scalars()
    x = eng.get_x()
    print("round x err", np.max(np.abs(x - (x0 - p_ref))) / np.max(np.abs(x0 - p_ref)), "shift err", abs(sc["shift_mean"] - shift) / shift)
