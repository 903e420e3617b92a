"""Diagnostic: run c0 rounds one at a time and check every client's TopK
delta against the oracle's compress of the device's own difference."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import fednl_oracle as O
from paper_2410_08760_b200 import data as D
from paper_2410_08760_b200.engine import FedNLEngine
name = sys.argv[1] if len(sys.argv) > 1 else "c0"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 120
shards = D.baseline_shards(name)
cfg = D.baseline_run_config(name, rounds=R)
d = shards[0].dim
eng = FedNLEngine(cfg, d, len(shards), shards[0].n_samples, lam=shards[0].lam)
eng.upload([s.bmat for s in shards])
eng.init_state()
k = cfg.compressor.k
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
if skip:
    eng.run_rounds(skip)
for r in range(skip, R):
    b = eng.run_rounds(1)
    bad = []
    nz = []
    for cid in range(len(shards)):
        diff = eng.round_diff(cid)
        want = O.compress_packed(diff, d, "topk", k, O.round_stream(cfg.run_seed, cid, r))
        idx, val = eng.round_delta(cid)
        nz.append(int(np.count_nonzero(diff)))
        if not (np.array_equal(idx, want.indices) and np.array_equal(val, want.values)):
            bad.append((cid, len(idx), want.count, int(np.count_nonzero(diff))))
    print(r, "grad", b.grad_norm[0], "min/med nonzero", min(nz), int(np.median(nz)), "bad", bad[:6], flush=True)
    if bad:
        break
