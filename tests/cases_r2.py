"""Round-2 simulate cases shared by the CPU oracle pins and the GPU parity
tests (golden rows in tests/golden/simulate_r2.npz, written by
oracle/make_golden.py gen_sim_r2 from the reference itself).

* ls_deep / ls_deep8  FedNL-LS whose Armijo test backtracks 5..29 times in
                      every round (trial batches continue inside the round)
* ls_fail             LineSearchError after 61 trials (algorithms.py:311)
* ragged_*            shards of different n_i, each with its own lambda
                      (runtime.py:145-151 accepts them; oracle.py:33-46)
* c0_r20 / _mt        20 c0 rounds on 1 and 8 BLAS threads: the reference's
                      own run-to-run envelope
"""

from __future__ import annotations

import numpy as np

from paper_2410_08760_b200 import CompressorKind, CompressorSpec, RunConfig
from paper_2410_08760_b200 import data as D
from paper_2410_08760_b200.data import ClientShard

RAGGED_SIZES = (40, 23, 57, 31, 49)
RAGGED_LAMS = (1e-3, 2e-3, 3e-3, 4e-3, 5e-3)

SIM_R2 = {
    "ls_deep": (("synth", 8, 120, 4, 10), dict(rounds=8, algorithm="fednl-ls", kind="topk", k=9,
                                                ls_c=0.99, ls_gamma=0.9)),
    "ls_deep8": (("synth", 8, 120, 4, 10), dict(rounds=8, algorithm="fednl-ls", kind="topk", k=9,
                                                 ls_c=0.999, ls_gamma=0.5)),
    "ragged_topk": (("ragged", 7, RAGGED_SIZES, 21), dict(rounds=10, kind="topk", k=7)),
    "ragged_identity": (("ragged", 7, RAGGED_SIZES, 22), dict(rounds=8)),
    "ragged_exact": (("ragged", 7, RAGGED_SIZES, 23), dict(rounds=8, hessian_init="exact",
                                                           kind="randseqk", k=9)),
    "ragged_ls": (("ragged", 7, RAGGED_SIZES, 24), dict(rounds=8, algorithm="fednl-ls",
                                                        kind="toplek", k=9)),
    "ragged_pp": (("ragged", 7, RAGGED_SIZES, 25), dict(rounds=12, algorithm="fednl-pp", tau=2,
                                                        kind="randk", k=9)),
    "c0_r20": (("baseline", "c0"), dict(rounds=20)),
}
LS_FAIL = dict(base="ls_deep", ls_c=0.99, ls_gamma=0.97, rounds=4)


def ragged_shards(num_features: int, sizes, seed: int) -> list[ClientShard]:
    """One shuffled shard of sum(sizes) columns cut into consecutive pieces,
    lambdas cycling through RAGGED_LAMS (as make_golden.ragged_shards)."""
    (whole,) = D.make_shards(num_features, sum(sizes), 1, seed)
    out, lo = [], 0
    for i, sz in enumerate(sizes):
        out.append(ClientShard(bmat=np.asfortranarray(whole.bmat[:, lo:lo + sz]),
                               lam=RAGGED_LAMS[i % len(RAGGED_LAMS)]))
        lo += sz
    return out


def case_r2(name: str) -> tuple[dict, list[ClientShard]]:
    """(RunConfig keyword dict with kind / k, shards) of a round-2 case."""
    gen, kw = SIM_R2[name]
    kw = dict(kw)
    if gen[0] == "synth":
        _, nf, m, n, seed = gen
        shards = D.make_shards(nf, m, n, seed)
        kw.setdefault("run_seed", seed)
    elif gen[0] == "ragged":
        _, nf, sizes, seed = gen
        shards = ragged_shards(nf, sizes, seed)
        kw.setdefault("run_seed", seed)
    else:
        c = D.BASELINE_CONFIGS[gen[1]]
        shards = D.baseline_shards(gen[1])
        kw.setdefault("run_seed", 1)
        for key in ("algorithm", "kind", "k", "alpha", "tau"):
            if key in c:
                kw.setdefault(key, c[key])
    return kw, shards


def run_config(kw: dict) -> RunConfig:
    kw = dict(kw)
    kind = kw.pop("kind", "identity")
    k = kw.pop("k", None)
    return RunConfig(compressor=CompressorSpec(CompressorKind(kind), k=k), **kw)
