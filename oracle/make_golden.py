"""Generate tests/golden/*.npz from the REFERENCE itself (build container only).

Imports the read-only reference package from /root/reference/pkg/src and
records its outputs on fixed, seeded inputs.  The fixtures pin
`oracle/fednl_oracle.py` (tests/test_oracle_golden.py) and are the targets of
the GPU parity tests.  /root/reference does not exist on the GPU box, so the
vectors are committed.  Run:

    OPENBLAS_NUM_THREADS=1 python oracle/make_golden.py

Every fixture is small (the whole directory stays well under 2 MB).
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")

sys.path.insert(0, REF)
from fednl import linalg, oracle, rng  # noqa: E402
from fednl.algorithms import RunConfig  # noqa: E402
from fednl.compressors import CompressorKind, CompressorSpec, compress  # noqa: E402
from fednl.data import (  # noqa: E402
    RawDataset,
    augment_and_shard,
    generate_synthetic,
    normalize_labels,
)
from fednl.algorithms import LineSearchError  # noqa: E402
from fednl.oracle import ClientShard  # noqa: E402
from fednl.runtime import simulate  # noqa: E402

# The BASELINE configs; the shapes are used at reduced rounds.
BASELINE = {
    "c0": dict(d=301, n=142, ni=350, density=0.04, p_pos=0.3, lam=1e-3,
               algorithm="fednl", kind="topk", k=2408, alpha=1.0, rounds=100),
    "c1": dict(d=124, n=80, ni=407, density=0.11, p_pos=0.24, lam=1e-3,
               algorithm="fednl", kind="randseqk", k=992, alpha=None, rounds=200),
    "c2": dict(d=69, n=100, ni=110, density=0.44, p_pos=0.5, lam=1e-3,
               algorithm="fednl-ls", kind="toplek", k=69, alpha=None, rounds=200),
    "c3": dict(d=301, n=142, ni=350, density=0.04, p_pos=0.3, lam=1e-3,
               algorithm="fednl-pp", kind="randk", k=301, alpha=None, rounds=500, tau=12),
}


def binary_raw(num_features: int, m: int, density: float, p_pos: float, seed: int) -> RawDataset:
    """SURVEY §8(d) binary generator built with the reference's own Prg."""
    prg = rng.Prg(seed)
    feats = prg.f64_block(m * num_features).reshape(m, num_features) < density
    labels = np.where(prg.f64_block(m) < p_pos, 1.0, -1.0)
    rows = []
    for j in range(m):
        nz = np.flatnonzero(feats[j])
        rows.append((nz.astype(np.int64) + 1, np.ones(len(nz))))
    return RawDataset(labels=labels, rows=rows, num_features=num_features)


def baseline_shards(name: str, seed: int = 1):
    c = BASELINE[name]
    ds = binary_raw(c["d"] - 1, c["n"] * c["ni"], c["density"], c["p_pos"], seed)
    return augment_and_shard(ds, c["n"], run_seed=seed, lam=c["lam"])


def make_shards(num_features, m, n, seed, lam=1e-3):
    ds = generate_synthetic(num_features, m, seed=seed)
    normalize_labels(ds)
    return augment_and_shard(ds, n, run_seed=seed, lam=lam)


def rows_arrays(rows):
    return dict(
        round=np.array([r.round for r in rows], dtype=np.int64),
        grad_norm=np.array([r.grad_norm for r in rows]),
        f_value=np.array([r.f_value for r in rows]),
        bytes_up=np.array([r.bytes_up_cum for r in rows], dtype=np.int64),
        bytes_down=np.array([r.bytes_down_cum for r in rows], dtype=np.int64),
        ls_steps=np.array([r.ls_steps for r in rows], dtype=np.int64),
    )


def gen_rng():
    out = {}
    p = rng.Prg(0)
    out["seed0_stream"] = np.array([p.next_u64() for _ in range(5)], dtype=np.uint64)
    seeds = [0, 1, 42, 0xDEADBEEF, (1 << 64) - 1, 0x9E3779B97F4A7C15]
    out["stream_seeds"] = np.array(seeds, dtype=np.uint64)
    out["streams"] = np.stack([rng.Prg(s).u64_block(64) for s in seeds])
    out["f64_streams"] = np.stack([rng.Prg(s).f64_block(64) for s in seeds])
    bounds = [1, 2, 3, 10, 69, 80, 100, 131, 142, 2415, 7750, 45451, 524800,
              (1 << 63) + 12345, (1 << 64) - 1]
    out["rr_bounds"] = np.array(bounds, dtype=np.uint64)
    rr = np.zeros((len(seeds), len(bounds), 8), dtype=np.uint64)
    nxt = np.zeros((len(seeds), len(bounds)), dtype=np.uint64)
    for a, s in enumerate(seeds):
        for b, bd in enumerate(bounds):
            p = rng.Prg(s)
            rr[a, b] = [p.randrange(bd) for _ in range(8)]
            nxt[a, b] = p.next_u64()  # draw consumption check
    out["randrange"] = rr
    out["randrange_next"] = nxt
    # partial shuffles at the RandK and PP shapes
    ps = {}
    for key, (n, k, s) in {
        "randk_c3": (45451, 301, rng.derive_round_seed(1, 5, 7)),
        "pp_c3": (142, 12, rng.mix64(1 ^ rng.TAG_MASTER)),
        "small": (10, 4, 123),
        "full": (17, 17, 9),
    }.items():
        ps[key] = rng.Prg(s).partial_shuffle_prefix(n, k)
        out[f"pshuffle_{key}"] = ps[key]
        out[f"pshuffle_{key}_args"] = np.array([n, k, s], dtype=np.uint64)
    # the persistent master subset stream over 20 rounds (algorithms.py:422-425)
    mp = rng.derive_stream(1, rng.TAG_MASTER)
    out["pp_subsets_c3"] = np.stack(
        [np.sort(mp.partial_shuffle_prefix(142, 12)) for _ in range(20)]
    )
    grid = np.zeros((4, 6, 6), dtype=np.uint64)
    for a, rs in enumerate([0, 1, 123, (1 << 64) - 1]):
        for c in range(6):
            for r in range(6):
                grid[a, c, r] = rng.derive_round_seed(rs, c * 1000 + c, r * 77 + r)
    out["round_seed_grid"] = grid
    out["tags"] = np.array([rng.TAG_SHUFFLE, rng.TAG_SYNTH, rng.TAG_MASTER], dtype=np.uint64)
    return out


def compress_cases():
    """Packed inputs exercising ties, zeros, small/large k."""
    cases = []
    g = np.random.default_rng(2024)
    for d in (2, 3, 5, 9, 24):
        w = linalg.packed_length(d)
        a = g.standard_normal((d, d))
        cases.append((f"gauss{d}", d, linalg.pack_upper(np.asfortranarray((a + a.T) / 2))))
    for d in (7, 24, 40):
        w = linalg.packed_length(d)
        # quantised values: heavy ties across the k-th boundary, both signs
        v = g.integers(-3, 4, w).astype(float) * 0.125
        cases.append((f"ties{d}", d, v))
    cases.append(("onehot6", 6, np.eye(1, 21, 7).ravel() * -2.5))
    cases.append(("const5", 5, np.full(15, 0.75)))
    cases.append(("zeros4", 4, np.zeros(10)))
    # the round-0 difference of a real c2-shaped client (x = 0): Hessian - lam I
    sh = baseline_shards("c2")[3]
    x = np.zeros(sh.dim)
    s = oracle.new_scratch(sh)
    oracle.refresh_scratch(sh, x, s)
    h = oracle.hessian(sh, x, s)
    linalg.add_to_diagonal(h, -sh.lam)
    cases.append(("c2client3_round0", sh.dim, linalg.pack_upper(h)))
    return cases


def gen_compress():
    out = {}
    names = []
    for name, d, pk in compress_cases():
        w = linalg.packed_length(d)
        m = linalg.unpack_to_symmetric(np.asarray(pk, dtype=float), d)
        out[f"{name}__input"] = np.asarray(pk, dtype=float)
        out[f"{name}__d"] = np.array(d)
        names.append(name)
        ks = sorted({1, 2, max(1, w // 7), max(1, w // 2), w})
        for k in ks:
            for kind, weighted in (("topk", False), ("topk", True), ("toplek", False),
                                   ("randk", False), ("randseqk", False)):
                for seed in (0, 77, 0xABCDEF):
                    spec = CompressorSpec(CompressorKind(kind), k=k, topk_weighted=weighted)
                    prg = rng.Prg(seed)
                    delta = compress(m, spec, prg)
                    tag = f"{name}__{kind}{'W' if weighted else ''}__k{k}__s{seed}"
                    out[tag + "__idx"] = np.asarray(delta.indices, dtype=np.uint32)
                    out[tag + "__val"] = np.asarray(delta.values, dtype=float)
                    out[tag + "__next"] = np.array(prg.next_u64(), dtype=np.uint64)
                    if kind == "topk":
                        break  # deterministic: one seed is enough
        for kind in ("identity", "natural"):
            spec = CompressorSpec(CompressorKind(kind))
            prg = rng.Prg(5)
            delta = compress(m, spec, prg)
            tag = f"{name}__{kind}__s5"
            out[tag + "__val"] = np.asarray(delta.values, dtype=float)
            out[tag + "__next"] = np.array(prg.next_u64(), dtype=np.uint64)
    out["case_names"] = np.array(names)
    return out


def gen_oracle():
    out = {}
    shards = make_shards(6, 90, 3, seed=5, lam=0.01)
    g = np.random.default_rng(9)
    xs = [np.zeros(7), g.standard_normal(7), 30.0 * g.standard_normal(7)]
    for ci, sh in enumerate(shards):
        out[f"bmat{ci}"] = np.asfortranarray(sh.bmat)
        for xi, x in enumerate(xs):
            s = oracle.new_scratch(sh)
            oracle.refresh_scratch(sh, x, s)
            out[f"f_{ci}_{xi}"] = np.array(oracle.f_value(sh, x, s))
            out[f"grad_{ci}_{xi}"] = oracle.gradient(sh, x, s)
            out[f"hess_{ci}_{xi}"] = linalg.pack_upper(oracle.hessian(sh, x, s))
    out["xs"] = np.stack(xs)
    out["lam"] = np.array(0.01)
    return out


def gen_linalg():
    out = {}
    g = np.random.default_rng(31)
    for d in (1, 2, 10, 50, 301):
        a = g.standard_normal((d, d))
        spd = np.asfortranarray(a @ a.T / d + np.eye(d))
        b = g.standard_normal(d)
        out[f"spd{d}"] = linalg.pack_upper(spd)
        out[f"rhs{d}"] = b
        out[f"sol{d}"] = linalg.cholesky_solve(spd, b)
    bad = np.asfortranarray([[1.0, 2.0], [2.0, 1.0]])
    try:
        linalg.cholesky_factor(bad)
    except linalg.NotPositiveDefiniteError as e:
        out["npd_pk"] = linalg.pack_upper(bad)
        out["npd_pivot"] = np.array([e.pivot_index, e.pivot_value])
    a = g.standard_normal((12, 12))
    ind = np.asfortranarray(a @ a.T)
    ind[7, 7] = -50.0
    try:
        linalg.cholesky_factor(ind)
    except linalg.NotPositiveDefiniteError as e:
        out["npd2_pk"] = linalg.pack_upper(ind)
        out["npd2_pivot"] = np.array([e.pivot_index, e.pivot_value])
    return out


def gen_eigen():
    """jacobi_eigh / eigen_clamp_min (linalg.py:189-259) of random symmetric,
    indefinite, diagonal and repeated-eigenvalue matrices."""
    out = {}
    g = np.random.default_rng(57)
    mats = {}
    for d in (1, 2, 5, 20, 60):
        a = g.standard_normal((d, d))
        mats[f"sym{d}"] = (a + a.T) / 2.0
    mats["diag3"] = np.diag([3.0, -1.0, 2.0])
    q, _ = np.linalg.qr(g.standard_normal((9, 9)))
    mats["rep9"] = (q * np.array([-2.0, -2.0, -2.0, 0.1, 0.1, 1.0, 1.0, 1.0, 5.0])) @ q.T
    a = g.standard_normal((30, 30))
    mats["spd30"] = a @ a.T / 30.0 + np.eye(30)
    for name, m in mats.items():
        m = np.asfortranarray(m)
        vals, vecs = linalg.jacobi_eigh(m.copy(order="F"))
        out[f"{name}__pk"] = linalg.pack_upper(m)
        out[f"{name}__vals_sorted"] = np.sort(vals)
        for floor in (0.5, 1e-12):
            out[f"{name}__clamp{floor:g}"] = linalg.pack_upper(linalg.eigen_clamp_min(m, floor))
    out["names"] = np.array(sorted(mats))
    return out


SIM_CASES = {
    # name: (generator args, RunConfig kwargs)
    "fednl_identity": (("synth", 6, 80, 4, 2), dict(rounds=12)),
    "fednl_topk": (("synth", 8, 120, 5, 3), dict(rounds=10, compressor=("topk", 9))),
    "fednl_topkW": (("synth", 8, 120, 5, 3), dict(rounds=10, compressor=("topk", 9, True))),
    "fednl_toplek": (("synth", 8, 120, 5, 4), dict(rounds=10, compressor=("toplek", 9))),
    "fednl_randk": (("synth", 8, 120, 5, 5), dict(rounds=10, compressor=("randk", 9))),
    "fednl_randseqk": (("synth", 8, 120, 5, 6), dict(rounds=10, compressor=("randseqk", 9))),
    "fednl_natural": (("synth", 8, 120, 5, 7), dict(rounds=8, compressor=("natural",))),
    "fednl_alpha1_stop": (("synth", 5, 60, 2, 6), dict(rounds=50, alpha=1.0,
                                                         compressor=("topk", 4), stop_grad_norm=1e-9)),
    "fednl_zero_init": (("synth", 6, 80, 4, 8), dict(rounds=6, hessian_init="zero",
                                                       compressor=("topk", 8))),
    "fednl_exact_init": (("synth", 6, 80, 4, 9), dict(rounds=6, hessian_init="exact",
                                                        compressor=("randseqk", 8))),
    "ls_topk": (("synth", 8, 120, 4, 10), dict(rounds=10, algorithm="fednl-ls", compressor=("topk", 9))),
    "ls_toplek": (("synth", 8, 120, 4, 11), dict(rounds=10, algorithm="fednl-ls",
                                                  compressor=("toplek", 12))),
    "pp_randk": (("synth", 8, 150, 6, 12), dict(rounds=15, algorithm="fednl-pp", tau=2,
                                                 compressor=("randk", 9))),
    "pp_topk": (("synth", 8, 150, 6, 13), dict(rounds=15, algorithm="fednl-pp", tau=3,
                                                compressor=("topk", 9))),
    "pp_identity_stop": (("synth", 4, 60, 4, 8), dict(rounds=60, algorithm="fednl-pp", tau=2,
                                                       stop_grad_norm=1e-10)),
    # option a (eigen_clamp_min of the estimate, algorithms.py:361-364)
    "fednl_opt_a": (("synth", 8, 120, 5, 14), dict(rounds=10, option="a", compressor=("topk", 9))),
    "fednl_opt_a_mu": (("synth", 8, 120, 5, 15), dict(rounds=10, option="a", mu=0.05,
                                                       compressor=("randseqk", 9))),
    "ls_opt_a": (("synth", 8, 120, 4, 16), dict(rounds=10, algorithm="fednl-ls", option="a",
                                                 mu=0.02, compressor=("toplek", 12))),
    # BASELINE shapes at reduced round counts
    "c0_r4": (("baseline", "c0"), dict(rounds=4)),
    "c1_r30": (("baseline", "c1"), dict(rounds=30)),
    "c2_r30": (("baseline", "c2"), dict(rounds=30)),
    "c3_r30": (("baseline", "c3"), dict(rounds=30)),
}


def build_case(name):
    gen, kw = SIM_CASES[name]
    kw = dict(kw)
    if gen[0] == "synth":
        _, nf, m, n, seed = gen
        shards = make_shards(nf, m, n, seed)
        kw.setdefault("run_seed", seed)
    else:
        c = BASELINE[gen[1]]
        shards = baseline_shards(gen[1], seed=1)
        kw.setdefault("run_seed", 1)
        kw.setdefault("algorithm", c["algorithm"])
        kw.setdefault("compressor", (c["kind"], c["k"]))
        kw.setdefault("alpha", c["alpha"])
        if "tau" in c:
            kw.setdefault("tau", c["tau"])
    comp = kw.pop("compressor", ("identity",))
    spec = CompressorSpec(CompressorKind(comp[0]), k=comp[1] if len(comp) > 1 else None,
                          topk_weighted=comp[2] if len(comp) > 2 else False)
    cfg = RunConfig(compressor=spec, **kw)
    return cfg, shards


def gen_sim(names=None):
    import threadpoolctl

    out = {}
    for name in names or [n for n in SIM_CASES if "opt_a" not in n]:
        cfg, shards = build_case(name)
        with threadpoolctl.threadpool_limits(1, "blas"):
            rows = simulate(cfg, shards)
        for k, v in rows_arrays(rows).items():
            out[f"{name}__{k}"] = v
        print(f"  sim {name}: {len(rows)} rows, final |g|={rows[-1].grad_norm:.3e}")
    if names is not None:
        return out
    # The reference's own envelope on the tie-heavy TopK shape: the same run
    # with 8 BLAS threads takes a different (equally valid) k-th-boundary
    # branch at round 3.  Both trajectories are recorded.
    cfg, shards = build_case("c0_r4")
    with threadpoolctl.threadpool_limits(8, "blas"):
        rows = simulate(cfg, shards)
    for k, v in rows_arrays(rows).items():
        out[f"c0_r4_mt__{k}"] = v
    return out


def gen_data():
    """Checksums of the reference's shards for every BASELINE shape (c0-c3)."""
    out = {}
    for name in ("c0", "c1", "c2"):
        shards = baseline_shards(name, seed=1)
        out[f"{name}__colsum"] = np.stack([s.bmat.sum(axis=0) for s in shards[:4]])
        out[f"{name}__rowsum"] = np.stack([s.bmat.sum(axis=1) for s in shards])
        out[f"{name}__first_col"] = np.stack([s.bmat[:, 0] for s in shards])
    sh = make_shards(6, 90, 3, seed=5, lam=0.01)
    out["synth_6_90_3_5"] = np.stack([s.bmat for s in sh])
    return out


def gen_topk_c0():
    """Round-0 TopK index sets of the first clients at the full c0 shape.

    At x = 0 every sigmoid is 1/2, so H_i - lam I has massive exact ties at
    the k-th boundary; the reference's lexsort tie rule decides them.
    """
    out = {}
    shards = baseline_shards("c0", seed=1)
    spec = CompressorSpec(CompressorKind.TOPK, k=2408)
    for cid in (0, 1, 77, 141):
        sh = shards[cid]
        x = np.zeros(sh.dim)
        s = oracle.new_scratch(sh)
        oracle.refresh_scratch(sh, x, s)
        h = oracle.hessian(sh, x, s)
        hest = linalg.new_matrix(sh.dim)
        linalg.add_to_diagonal(hest, sh.lam)
        delta = compress(h - hest, spec, rng.derive_round_prg(1, cid, 0))
        out[f"cid{cid}__idx"] = delta.indices
        out[f"cid{cid}__val"] = delta.values
    return out


INGEST_GOOD = (
    b"# comment line\n"
    b"+1 1:0.5 3:2 7:-1.25e-3\n"
    b"\n"
    b"-1\t2:1 3:1\r\n"
    b"  +1 4:3.0000000000000004   9:1e300\n"
    b"-1 1:-0 2:0.1\n"
    b"+1\n"
    b"-1 5:7 6:8 8:9\n"
    b"+1 1:1 2:2 3:3 4:4\n"
    b"   # indented comment\n"
    b"-1 9:0.3333333333333333\n"
)
INGEST_BAD = {
    "bad_label": b"+1 1:1\nabc 2:3\n",
    "three_labels": b"1 1:1\n2 1:1\n3 1:1\n",
    "no_colon": b"1 1:1\n0 2 3:1\n",
    "bad_index": b"1 x:1\n",
    "index_zero": b"1 0:1\n",
    "not_increasing": b"1 3:1 3:2\n",
    "decreasing": b"1   5:1   2:2\n",
    "bad_value": b"1 1:1 2:abc\n",
    "empty": b"# only\n\n",
}


def gen_ingest():
    """LIBSVM parse / write / normalize / augment_and_shard / split_rows
    (data.py:31-254) on crafted inputs, and the ParseError positions."""
    from fednl.data import ParseError, parse_libsvm, split_rows, write_libsvm

    out = {}
    ds = parse_libsvm(INGEST_GOOD)
    out["good__labels"] = ds.labels
    out["good__num_features"] = np.array(ds.num_features)
    out["good__lens"] = np.array([len(r[0]) for r in ds.rows])
    out["good__idx"] = np.concatenate([r[0] for r in ds.rows])
    out["good__val"] = np.concatenate([r[1] for r in ds.rows])
    out["good__written"] = np.frombuffer(write_libsvm(ds), dtype=np.uint8)
    for name, buf in INGEST_BAD.items():
        try:
            parse_libsvm(buf)
            raise AssertionError(name)
        except ParseError as e:
            out[f"bad_{name}"] = np.array([e.line, e.col])
            out[f"bad_{name}__msg"] = np.array(str(e))
    for pair in ((0.0, 1.0), (-1.0, 1.0), (2.0, 7.0)):
        raw = RawDataset(labels=np.array([pair[1], pair[0], pair[1]]), rows=[(np.zeros(0, dtype=np.int64), np.zeros(0))] * 3, num_features=1)
        normalize_labels(raw)
        out[f"norm_{pair[0]:g}_{pair[1]:g}"] = raw.labels
    g = np.random.default_rng(3)
    rows, labels = [], []
    for i in range(23):
        nz = np.sort(g.choice(np.arange(1, 12), size=int(g.integers(0, 5)), replace=False))
        rows.append((nz.astype(np.int64), g.standard_normal(len(nz))))
        labels.append(1.0 if g.random() < 0.4 else -1.0)
    big = RawDataset(labels=np.array(labels), rows=rows, num_features=11)
    out["shard__labels"] = big.labels
    out["shard__lens"] = np.array([len(r[0]) for r in rows])
    out["shard__idx"] = np.concatenate([r[0] for r in rows])
    out["shard__val"] = np.concatenate([r[1] for r in rows])
    shards = augment_and_shard(big, 4, 9, 0.01)
    out["shard__bmats"] = np.stack([s.bmat for s in shards])
    pieces = split_rows(big, 4, 9)
    out["shard__split_labels"] = np.stack([p.labels for p in pieces])
    return out


# ---- round-2 additions (simulate_r2.npz): line-search continuation and
# failure, ragged shards with per-shard lambda, a longer c0 trajectory with
# the reference's own 1- vs 8-thread envelope
SIM_R2 = {
    # Armijo with c close to 1 backtracks s = 5..29 times every round: the
    # trial batches continue past the first one inside every (mid-chunk) round
    "ls_deep": (("synth", 8, 120, 4, 10), dict(rounds=8, algorithm="fednl-ls", compressor=("topk", 9),
                                                ls_c=0.99, ls_gamma=0.9)),
    "ls_deep8": (("synth", 8, 120, 4, 10), dict(rounds=8, algorithm="fednl-ls", compressor=("topk", 9),
                                                 ls_c=0.999, ls_gamma=0.5)),
    # shards of 40 / 23 / 57 / 31 / 49 samples, lambdas 1e-3 .. 5e-3
    "ragged_topk": (("ragged", 7, (40, 23, 57, 31, 49), 21), dict(rounds=10, compressor=("topk", 7))),
    "ragged_identity": (("ragged", 7, (40, 23, 57, 31, 49), 22), dict(rounds=8)),
    "ragged_exact": (("ragged", 7, (40, 23, 57, 31, 49), 23), dict(rounds=8, hessian_init="exact",
                                                                      compressor=("randseqk", 9))),
    "ragged_ls": (("ragged", 7, (40, 23, 57, 31, 49), 24), dict(rounds=8, algorithm="fednl-ls",
                                                                   compressor=("toplek", 9))),
    "ragged_pp": (("ragged", 7, (40, 23, 57, 31, 49), 25), dict(rounds=12, algorithm="fednl-pp", tau=2,
                                                                   compressor=("randk", 9))),
    "c0_r20": (("baseline", "c0"), dict(rounds=20)),
}
RAGGED_LAMS = (1e-3, 2e-3, 3e-3, 4e-3, 5e-3)


def ragged_shards(num_features, sizes, seed):
    """One shuffled shard of sum(sizes) columns cut into consecutive pieces,
    each a ClientShard with its own lambda (the shape load_client_shard
    produces per client, data.py:236-254)."""
    (whole,) = make_shards(num_features, sum(sizes), 1, seed)
    out, lo = [], 0
    for i, sz in enumerate(sizes):
        out.append(ClientShard(bmat=np.asfortranarray(whole.bmat[:, lo:lo + sz]),
                               lam=RAGGED_LAMS[i % len(RAGGED_LAMS)]))
        lo += sz
    return out


def build_case_r2(name):
    gen, kw = SIM_R2[name]
    if gen[0] == "ragged":
        _, nf, sizes, seed = gen
        kw = dict(kw)
        kw.setdefault("run_seed", seed)
        comp = kw.pop("compressor", ("identity",))
        spec = CompressorSpec(CompressorKind(comp[0]), k=comp[1] if len(comp) > 1 else None)
        return RunConfig(compressor=spec, **kw), ragged_shards(nf, sizes, seed)
    SIM_CASES[name] = SIM_R2[name]
    try:
        return build_case(name)
    finally:
        del SIM_CASES[name]


def gen_sim_r2():
    import threadpoolctl

    out = {}
    for name in SIM_R2:
        cfg, shards = build_case_r2(name)
        with threadpoolctl.threadpool_limits(1, "blas"):
            rows = simulate(cfg, shards)
        for k, v in rows_arrays(rows).items():
            out[f"{name}__{k}"] = v
        print(f"  sim {name}: {len(rows)} rows, final |g|={rows[-1].grad_norm:.3e}, "
              f"ls {[r.ls_steps for r in rows]}")
    cfg, shards = build_case_r2("c0_r20")
    with threadpoolctl.threadpool_limits(8, "blas"):
        rows = simulate(cfg, shards)
    for k, v in rows_arrays(rows).items():
        out[f"c0_r20_mt__{k}"] = v
    # LineSearchError: Armijo c = 0.99 with gamma = 0.97 cannot pass in 61 trials
    cfg, shards = build_case_r2("ls_deep")
    cfg = RunConfig(compressor=cfg.compressor, rounds=4, algorithm="fednl-ls", ls_c=0.99,
                    ls_gamma=0.97, run_seed=cfg.run_seed)
    try:
        with threadpoolctl.threadpool_limits(1, "blas"):
            simulate(cfg, shards)
        raise AssertionError("expected LineSearchError")
    except LineSearchError as e:
        import re

        f_start, f_best = (float(v) for v in re.findall(r"f=([-0-9.eE+]+)", str(e)))
        out["ls_fail__round"] = np.array(e.round)
        out["ls_fail__f_start"] = np.array(f_start)
        out["ls_fail__f_best"] = np.array(f_best)
        out["ls_fail__message"] = np.array(str(e))
        print(f"  ls_fail: {e}")
    return out


def gaussian_shards_c4(d=1024, n=512, ni=2048, lam=1e-4, seed=1):
    """SURVEY §8(d) c4 generator (numpy default_rng), as
    paper_2410_08760_b200.data.gaussian_shards builds it, as reference
    ClientShards."""
    g = np.random.default_rng(seed)
    wstar = g.standard_normal(d - 1) / np.sqrt(d)
    out = []
    for _ in range(n):
        a = g.standard_normal((d - 1, ni))
        y = np.sign(wstar @ a + g.normal(0.0, np.sqrt(0.1), ni))
        y[y == 0] = 1.0
        b = np.empty((d, ni), order="F")
        b[: d - 1] = a
        b[d - 1] = 1.0
        b *= y
        out.append(ClientShard(bmat=b, lam=lam))
    return out


def gen_c4():
    """Two c4 rounds (d=1024, n=512, n_i=2048, TopK k=8192, lambda=1e-4) from
    the reference simulate (8 worker threads, 1 BLAS thread each: the rows do
    not depend on the worker count, runtime.py:141-143)."""
    import threadpoolctl

    shards = gaussian_shards_c4()
    cfg = RunConfig(compressor=CompressorSpec(CompressorKind.TOPK, k=8192), rounds=2, lam=1e-4, run_seed=1)
    with threadpoolctl.threadpool_limits(1, "blas"):
        rows = simulate(cfg, shards, workers=8)
    out = {f"c4_r2__{k}": v for k, v in rows_arrays(rows).items()}
    print(f"  c4: {len(rows)} rows, |g| {[r.grad_norm for r in rows]}")
    return out


def gen_compress_r2():
    """Compressors past the one-CTA envelope of round 1: TopLEK at w = 45,451
    (d = 301: the paper's W8A TopLEK[8d] shape) on tie-heavy round-0 c0
    differences and on Gaussian inputs; RandK with k > 6000."""
    out = {}
    shards = baseline_shards("c0")
    d = shards[0].dim
    x = np.zeros(d)
    g = np.random.default_rng(99)
    inputs = {}
    for cid in (0, 5, 77):
        sh = shards[cid]
        s = oracle.new_scratch(sh)
        oracle.refresh_scratch(sh, x, s)
        h = oracle.hessian(sh, x, s)
        linalg.add_to_diagonal(h, -sh.lam)
        inputs[f"c0client{cid}_round0"] = linalg.pack_upper(h)
    a = g.standard_normal((d, d))
    inputs["gauss301"] = linalg.pack_upper(np.asfortranarray((a + a.T) / 2))
    names = sorted(inputs)
    for name in names:
        pk = inputs[name]
        out[f"{name}__input"] = pk
        m = linalg.unpack_to_symmetric(pk, d)
        for kind, k in (("toplek", 301), ("toplek", 2408), ("toplek", 20000), ("randk", 8000),
                        ("randk", 30000)):
            for seed in (3, 0xC0FFEE):
                prg = rng.Prg(seed)
                delta = compress(m, CompressorSpec(CompressorKind(kind), k=k), prg)
                tag = f"{name}__{kind}__k{k}__s{seed}"
                out[tag + "__idx"] = np.asarray(delta.indices, dtype=np.uint32)
                out[tag + "__val"] = np.asarray(delta.values, dtype=float)
                out[tag + "__next"] = np.array(prg.next_u64(), dtype=np.uint64)
    out["names"] = np.array(names)
    out["d"] = np.array(d)
    # FedNL-LS with TopLEK[8d] on the c0 data (the W8A TopLEK run's shape)
    import threadpoolctl

    cfg = RunConfig(algorithm="fednl-ls", compressor=CompressorSpec(CompressorKind.TOPLEK, k=8 * d),
                    rounds=6, run_seed=1)
    with threadpoolctl.threadpool_limits(1, "blas"):
        rows = simulate(cfg, shards)
    for k2, v in rows_arrays(rows).items():
        out[f"ls_toplek8d_c0__{k2}"] = v
    print(f"  ls_toplek8d_c0: |g| {[r.grad_norm for r in rows]}")
    return out


def gen_csv():
    """The reference's metrics CSV text and canonical_config lines
    (runtime.py:69-113, transport.py:205-232) for fixed rows and configs."""
    import io

    from fednl.runtime import MetricsRow, write_csv
    from fednl.transport import canonical_config

    rows = [MetricsRow(0, 0.0, 0.24282060357349974, 0.6931471805599453, 0, 42784, 0),
            MetricsRow(1, 0.012345678901234568, 1e-300, -0.0, 31312, 85568, 3),
            MetricsRow(2, 1.5, 5e-324, 1.7976931348623157e308, 2**40, 2**41, 60)]
    out = {}
    cfgs = {
        "default": RunConfig(),
        "c0": RunConfig(compressor=CompressorSpec(CompressorKind.TOPK, k=2408), alpha=1.0, rounds=100, run_seed=1),
        "ls": RunConfig(algorithm="fednl-ls", compressor=CompressorSpec(CompressorKind.TOPLEK, k=69),
                        ls_c=0.3, ls_gamma=0.7, lam=1e-4),
        "pp": RunConfig(algorithm="fednl-pp", tau=12, compressor=CompressorSpec(CompressorKind.RANDK, k=301),
                        reconstruct_indices=False, hessian_init="exact", run_seed=2**40),
        "opt_a": RunConfig(option="a", mu=0.05, compressor=CompressorSpec(CompressorKind.TOPK, k=9,
                                                                            topk_weighted=True)),
        "natural": RunConfig(compressor=CompressorSpec(CompressorKind.NATURAL), hessian_init="zero"),
    }
    names = sorted(cfgs)
    for name in names:
        line = canonical_config(cfgs[name], 301 if name != "ls" else 69, 142)
        buf = io.StringIO()
        write_csv(rows, buf, config_line=line)
        out[f"{name}__line"] = np.array(line)
        out[f"{name}__csv"] = np.array(buf.getvalue())
    buf = io.StringIO()
    write_csv(rows, buf)
    out["noconfig__csv"] = np.array(buf.getvalue())
    out["names"] = np.array(names)
    return out


FULL_CASES = {  # the BASELINE configs' full round counts
    "c0_full": (("baseline", "c0"), dict(rounds=100)),
    "c1_full": (("baseline", "c1"), dict(rounds=200)),
    "c2_full": (("baseline", "c2"), dict(rounds=200)),
    "c3_full": (("baseline", "c3"), dict(rounds=500)),
}


def gen_full():
    """Whole BASELINE runs of c1 / c2 / c3 from the reference's simulate on 1
    and on 8 BLAS threads (two equally valid trajectories: the row check
    accepts either)."""
    import threadpoolctl

    out = {}
    for name, (gen, kw) in FULL_CASES.items():
        SIM_CASES[name] = (gen, kw)
        cfg, shards = build_case(name)
        for threads, tag in ((1, name), (8, name + "_mt")):
            with threadpoolctl.threadpool_limits(threads, "blas"):
                rows = simulate(cfg, shards)
            for k, v in rows_arrays(rows).items():
                out[f"{tag}__{k}"] = v
            print(f"  full {tag}: {len(rows)} rows, final |g|={rows[-1].grad_norm:.3e}")
    return out


def gen_sim_opt_a():
    return gen_sim([n for n in SIM_CASES if "opt_a" in n])


def main(only=None):
    os.makedirs(OUT, exist_ok=True)
    for fname, fn in (
        ("rng.npz", gen_rng),
        ("compress.npz", gen_compress),
        ("oracle.npz", gen_oracle),
        ("linalg.npz", gen_linalg),
        ("data.npz", gen_data),
        ("topk_c0_round0.npz", gen_topk_c0),
        ("simulate.npz", gen_sim),
        ("eigen.npz", gen_eigen),
        ("simulate_opt_a.npz", gen_sim_opt_a),
        ("ingest.npz", gen_ingest),
        ("simulate_r2.npz", gen_sim_r2),
        ("simulate_c4.npz", gen_c4),
        ("compress_r2.npz", gen_compress_r2),
        ("csv.npz", gen_csv),
        ("simulate_full.npz", gen_full),
    ):
        if only and fname not in only:
            continue
        print(f"generating {fname}")
        np.savez_compressed(os.path.join(OUT, fname), **fn())
    for f in sorted(os.listdir(OUT)):
        print(f"{f}: {os.path.getsize(os.path.join(OUT, f))} bytes")


if __name__ == "__main__":
    main(sys.argv[1:] or None)
