"""Diagnostic: the c0 round-0 differences (massive exact ties) of all 142
clients through the split TopK (forced), three times, against the oracle."""
import os, sys
os.environ.setdefault("FB_TOPK_SPLIT", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import fednl_oracle as O
from paper_2410_08760_b200 import data as D, leaf, CompressorSpec, CompressorKind
shards = D.baseline_shards("c0")
d = shards[0].dim
P = []
for s in shards:
    ev = O.local_eval(s.bmat, 1e-3, np.zeros(d))
    diff = ev.hess.copy()
    diff[O.diag_positions(d)] -= 1e-3
    P.append(diff)
P = np.stack(P)
seeds = [O.round_seed(1, c, 0) for c in range(len(shards))]
want = [O.compress_packed(P[c], d, "topk", 2408, O.SplitMix64(seeds[c])) for c in range(len(shards))]
for rep in range(3):
    got = leaf.compress_packed_batch(P, d, CompressorSpec(CompressorKind.TOPK, k=2408), seeds)
    bad = [(c, got[c].entry_count, len(np.setdiff1d(want[c].indices, got[c].indices)))
           for c in range(len(shards)) if not np.array_equal(got[c].indices, want[c].indices)]
    print("rep", rep, "bad clients", len(bad), bad[:8], flush=True)
