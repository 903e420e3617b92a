"""CUDA path vs the pinned CPU oracle and the reference's golden vectors.

Protocol:
  P0 PRNG            bit-exact
  P1 compressors     bit-exact indices / values / counts / draws on identical inputs
  P2 oracle          normwise 1e-10 per client and quantity
  P3 shift + fold    bit-exact given identical deltas
  P4 solve           1e-10 relative; same pivot index on failure
  P6 trajectories    1e-10 with a floor for data-independent selectors;
                     TopK / TopLEK within the reference's own envelope
All calls go through the C ABI (libfednl_b200.so).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from oracle import fednl_oracle as O
from paper_2410_08760_b200 import (
    CompressorKind,
    CompressorSpec,
    NotPositiveDefiniteError,
    RunConfig,
    leaf,
    simulate,
)
from paper_2410_08760_b200 import _lib
from paper_2410_08760_b200 import data as D
from paper_2410_08760_b200.engine import FedNLEngine

pytestmark = pytest.mark.gpu


def normwise(got, want, scale=None):
    want = np.asarray(want)
    s = np.max(np.abs(want)) if scale is None else scale
    return float(np.max(np.abs(np.asarray(got) - want))) / max(s, 1e-300)


# --------------------------------------------------------------------- P0


def test_device_prg_streams_match_golden():
    g = golden("rng.npz")
    assert leaf.prg_u64(0, 5).tolist() == g["seed0_stream"].tolist()
    for a, s in enumerate(g["stream_seeds"].tolist()):
        assert np.array_equal(leaf.prg_u64(s, 64), g["streams"][a])


def test_device_randrange_and_consumption():
    g = golden("rng.npz")
    for a, s in enumerate(g["stream_seeds"].tolist()):
        out, nxt = leaf.prg_randrange(s, g["rr_bounds"].tolist(), 8)
        assert np.array_equal(out, g["randrange"][a])
        assert np.array_equal(nxt, g["randrange_next"][a])


def test_device_partial_shuffle_and_round_seeds():
    g = golden("rng.npz")
    for key in ("randk_c3", "pp_c3", "small", "full"):
        n, k, s = (int(v) for v in g[f"pshuffle_{key}_args"])
        assert np.array_equal(leaf.prg_partial_shuffle(s, n, k), g[f"pshuffle_{key}"])
    for a, rs in enumerate([0, 1, 123, (1 << 64) - 1]):
        for r in range(6):
            seeds = leaf.round_seeds(rs, 3, r)
            assert seeds.tolist() == [O.round_seed(rs, c, r) for c in range(3)]


# --------------------------------------------------------------------- P1


@pytest.fixture(params=["0", "1"], ids=["stream", "split"])
def topk_path(request, monkeypatch):
    """Both large-w TopK paths: the one-CTA-per-client k_topk_stream and the
    window / segmented pass / select kernels (chosen per context at creation;
    fb_config.topk_path pins either)."""
    path = _lib.TOPK_PATH_SPLIT if request.param == "1" else _lib.TOPK_PATH_STREAM
    monkeypatch.setattr(leaf, "TOPK_PATH", path)
    yield request.param


def _golden_compress_cases():
    g = golden("compress.npz")
    for name in g["case_names"].tolist():
        pk = g[f"{name}__input"]
        d = int(g[f"{name}__d"])
        for key in g.files:
            if key.startswith(name + "__") and key.endswith("__val"):
                tag = key[len(name) + 2:-5]
                yield g, name, d, pk, tag


def test_compressors_bit_exact_on_golden_inputs():
    n_checked = 0
    for g, name, d, pk, tag in _golden_compress_cases():
        parts = tag.split("__")
        kind = parts[0]
        weighted = kind.endswith("W")
        kind = kind.rstrip("W")
        if kind in ("identity", "natural"):
            k, seed = None, int(parts[1][1:])
        else:
            k, seed = int(parts[1][1:]), int(parts[2][1:])
        spec = CompressorSpec(CompressorKind(kind), k=k, topk_weighted=weighted)
        delta = leaf.compress_packed_batch(pk[None, :], d, spec, [seed])[0]
        base = f"{name}__{tag}"
        assert np.array_equal(delta.values, g[base + "__val"]), base
        if base + "__idx" in g.files:
            assert np.array_equal(delta.indices, g[base + "__idx"]), base
        # draw consumption: the next draw after compressing equals the reference's
        p = O.SplitMix64(seed)
        for _ in range(delta.draws):
            p.next_u64()
        assert p.next_u64() == int(g[base + "__next"]), base
        n_checked += 1
    assert n_checked > 300


def test_topk_round0_full_c0_shape_ties(topk_path):
    g = golden("topk_c0_round0.npz")
    shards = D.baseline_shards("c0")
    d = shards[0].dim
    cids = [0, 1, 77, 141]
    diffs = []
    for cid in cids:
        ev = O.local_eval(shards[cid].bmat, 1e-3, np.zeros(d))
        diff = ev.hess.copy()
        diff[O.diag_positions(d)] -= 1e-3
        diffs.append(diff)
    seeds = [O.round_seed(1, cid, 0) for cid in cids]
    deltas = leaf.compress_packed_batch(np.stack(diffs), d, CompressorSpec(CompressorKind.TOPK, k=2408), seeds)
    for cid, delta in zip(cids, deltas):
        assert np.array_equal(delta.indices, g[f"cid{cid}__idx"])
        assert np.array_equal(delta.values, g[f"cid{cid}__val"])


@pytest.mark.parametrize("kind,k", [("topk", 2408), ("randseqk", 2408), ("randk", 301), ("topk", 45451)])
def test_compressors_bit_exact_at_c0_size(kind, k, topk_path):
    """Random and tie-heavy inputs at w = 45451 against the oracle."""
    d = 301
    w = O.packed_len(d)
    rng = np.random.default_rng(7)
    P = rng.standard_normal((9, w))
    P[1] = np.round(P[1] * 4) / 4  # massive ties
    P[2] = 0.0  # empty delta
    P[3, ::3] = 0.0
    P[4] = np.abs(P[4])
    P[5] = -0.0 * P[5]  # negative zeros only -> all-zero
    # zeros complete the set (converged / structurally zero entries), with and
    # without subnormal keys above them; subnormals deciding the selection
    P[6] = 0.0
    P[6, rng.choice(w, 100, replace=False)] = rng.standard_normal(100)
    P[7] = 0.0
    P[7, rng.choice(w, 80, replace=False)] = np.concatenate([rng.standard_normal(50), rng.standard_normal(30) * 1e-310])
    P[8] = 0.0
    P[8, rng.choice(w, 3000, replace=False)] = np.concatenate([rng.standard_normal(2000), rng.standard_normal(1000) * 1e-310])
    seeds = [O.round_seed(9, c, 4) for c in range(len(P))]
    spec = CompressorSpec(CompressorKind(kind), k=k)
    got = leaf.compress_packed_batch(P, d, spec, seeds)
    for c in range(len(P)):
        want = O.compress_packed(P[c], d, kind, k, O.SplitMix64(seeds[c]))
        assert got[c].entry_count == want.count, c
        assert np.array_equal(got[c].indices, want.indices), c
        assert np.array_equal(got[c].values, want.values), c


@pytest.mark.parametrize("k", [8192, 1, 524800])
def test_topk_streaming_path_bit_exact_at_c4_size(k, topk_path):
    """w = 524,800 (c4) runs the streaming TopK (keys do not fit in shared
    memory): candidate path, exact-tie path, zero ties, take-all."""
    d = 1024
    w = O.packed_len(d)
    rng = np.random.default_rng(23)
    P = rng.standard_normal((7, w))
    P[1] = np.round(P[1] * 4) / 4  # few distinct values: huge exact-tie bins
    P[2] = 0.0  # empty delta
    P[3, ::3] = 0.0
    P[4] = 1.0 + rng.random(w)  # one exponent: the candidate list decides
    P[5] = 0.0
    P[5, rng.choice(w, 100, replace=False)] = rng.standard_normal(100)  # zeros complete the set
    P[6] = P[0] * 1e-300  # subnormal-heavy keys
    seeds = [O.round_seed(3, c, 1) for c in range(7)]
    got = leaf.compress_packed_batch(P, d, CompressorSpec(CompressorKind.TOPK, k=k), seeds)
    for c in range(7):
        want = O.compress_packed(P[c], d, "topk", k, O.SplitMix64(seeds[c]))
        assert got[c].entry_count == want.count, c
        assert np.array_equal(got[c].indices, want.indices), c
        assert np.array_equal(got[c].values, want.values), c


def test_topk_split_path_fallbacks_and_scratch_reuse(topk_path):
    """c4-like batch (n*w large enough that a segment's candidate slots are
    fewer than its positions): window miss (the strided sample sees only the
    small keys), a segment overflowing its candidate slots (one tie bin holds
    every key), tie bins beyond the select kernel's shared-memory list, zeros
    completing the set.  The same engine compresses the batch twice in
    different client orders: the tie/zero scratch rows must come back clean."""
    d = 1024
    w = O.packed_len(d)
    n = 80
    k = 8192
    rng = np.random.default_rng(31)
    P = rng.standard_normal((n, w))
    i = np.arange(8192)  # the window kernel's sample positions (tks_sample_pos)
    ts = (i // 8) * (w - 8) // 1024 + i % 8
    P[1] = 5.0 + rng.random(w)
    P[1, ts] = 1e-3
    P[2] = 1.0
    P[3] = np.round(P[3] * 4) / 4
    P[4] = 0.0
    P[4, rng.choice(w, 50, replace=False)] = 1.0
    P[5] *= rng.random(w) < 0.5
    P[6] = 0.0
    spec = CompressorSpec(CompressorKind.TOPK, k=k)
    check = list(range(8)) + [n - 2, n - 1]
    for order in (np.arange(n), np.arange(n)[::-1]):
        Q = np.ascontiguousarray(P[order])
        seeds = [O.round_seed(5, int(c), 2) for c in order]
        got = leaf.compress_packed_batch(Q, d, spec, seeds)
        for slot, c in enumerate(order):
            if c not in check:
                continue
            want = O.compress_packed(P[c], d, "topk", k, O.SplitMix64(seeds[slot]))
            assert got[slot].entry_count == want.count, c
            assert np.array_equal(got[slot].indices, want.indices), c
            assert np.array_equal(got[slot].values, want.values), c
    # c0 shape (w = 45,451 is not a multiple of the select kernel's block):
    # window misses both ways, converged-regime zero completion
    d = 301
    w = O.packed_len(d)
    i = np.arange(2048)
    ts = (i // 8) * (w - 8) // 256 + i % 8
    P = rng.standard_normal((6, w))
    P[0] = 5.0 + rng.random(w)
    P[0, ts] = 1e-3  # G >= k
    P[1] = 1e-3 * rng.random(w)
    P[1, ts] = 5.0  # G + M < k
    P[2] = 0.0
    P[2, rng.choice(w, 3000, replace=False)] = rng.standard_normal(3000) * 1e-12
    P[3] = 0.0
    P[3, 7000:9500] = rng.standard_normal(2500)  # nonzeros clustered away from the sample
    P[4] = 0.0
    P[4, ts[::4]] = 1.0
    seeds = [O.round_seed(6, c, 9) for c in range(6)]
    for rep in range(2):
        got = leaf.compress_packed_batch(P, d, CompressorSpec(CompressorKind.TOPK, k=2408), seeds)
        for c in range(6):
            want = O.compress_packed(P[c], d, "topk", 2408, O.SplitMix64(seeds[c]))
            assert got[c].entry_count == want.count, (rep, c)
            assert np.array_equal(got[c].indices, want.indices), (rep, c)
            assert np.array_equal(got[c].values, want.values), (rep, c)


def test_randk_hash_pool_path_bit_exact():
    """w = 80,200 > RK_DIRECT_W: the swap chain runs over the hashed pool."""
    d = 400
    w = O.packed_len(d)
    rng = np.random.default_rng(5)
    P = rng.standard_normal((3, w))
    P[1] = 0.0
    seeds = [O.round_seed(11, c, 2) for c in range(3)]
    for k in (400, 6000):
        got = leaf.compress_packed_batch(P, d, CompressorSpec(CompressorKind.RANDK, k=k), seeds)
        for c in range(3):
            want = O.compress_packed(P[c], d, "randk", k, O.SplitMix64(seeds[c]))
            assert got[c].entry_count == want.count, (k, c)
            assert np.array_equal(got[c].indices, want.indices), (k, c)
            assert np.array_equal(got[c].values, want.values), (k, c)


def test_toplek_bit_exact_at_c2_size():
    d = 69
    w = O.packed_len(d)
    rng = np.random.default_rng(11)
    P = rng.standard_normal((8, w)) * np.exp(rng.standard_normal((8, w)) * 3)
    P[2] = np.round(P[2])
    seeds = [O.round_seed(1, c, 17) for c in range(8)]
    for k in (1, 69, 600, w):
        got = leaf.compress_packed_batch(P, d, CompressorSpec(CompressorKind.TOPLEK, k=k), seeds)
        for c in range(8):
            want = O.compress_packed(P[c], d, "toplek", k, O.SplitMix64(seeds[c]))
            assert np.array_equal(got[c].indices, want.indices), (k, c)
            assert np.array_equal(got[c].values, want.values), (k, c)


def test_compress_rejects_nonfinite():
    d = 5
    w = O.packed_len(d)
    P = np.ones((2, w))
    P[1, 3] = np.inf
    with pytest.raises(ValueError):
        leaf.compress_packed_batch(P, d, CompressorSpec(CompressorKind.TOPK, k=3), [1, 2])


# --------------------------------------------------------------------- P2


def test_oracle_against_golden_values():
    g = golden("oracle.npz")
    lam = float(g["lam"])
    shards = [D.ClientShard(bmat=np.asfortranarray(g[f"bmat{ci}"]), lam=lam) for ci in range(3)]
    for xi, x in enumerate(g["xs"]):
        f, grad, hess = leaf.oracle_eval(shards, x)
        for ci in range(3):
            assert normwise(f[ci], g[f"f_{ci}_{xi}"]) <= 1e-10
            assert normwise(grad[ci], g[f"grad_{ci}_{xi}"]) <= 1e-10
            assert normwise(hess[ci], g[f"hess_{ci}_{xi}"]) <= 1e-10


@pytest.mark.parametrize("name", ["c0", "c1", "c2"])
def test_oracle_at_baseline_shapes(name):
    shards = D.baseline_shards(name)
    d = shards[0].dim
    rng = np.random.default_rng(5)
    for x in (np.zeros(d), 0.3 * rng.standard_normal(d)):
        f, grad, hess = leaf.oracle_eval(shards, x)
        for c in (0, len(shards) // 2, len(shards) - 1):
            ev = O.local_eval(shards[c].bmat, shards[c].lam, x)
            assert normwise(f[c], ev.f) <= 1e-10
            assert normwise(grad[c], ev.grad) <= 1e-10
            assert normwise(hess[c], ev.hess) <= 1e-10


# --------------------------------------------------------------------- P4


def test_solve_against_golden():
    g = golden("linalg.npz")
    for d in (1, 2, 10, 50, 301):
        z = leaf.shifted_solve(g[f"spd{d}"], d, 0.0, g[f"rhs{d}"])
        assert normwise(z, g[f"sol{d}"]) <= 1e-10
    for key in ("npd", "npd2"):
        pk = g[f"{key}_pk"]
        d = int((np.sqrt(8 * len(pk) + 1) - 1) / 2)
        with pytest.raises(NotPositiveDefiniteError) as exc:
            leaf.shifted_solve(pk, d, 0.0, np.ones(d))
        assert exc.value.pivot_index == int(g[f"{key}_pivot"][0])
        assert exc.value.pivot_value == pytest.approx(float(g[f"{key}_pivot"][1]), rel=1e-9)


@pytest.mark.parametrize("d", [33, 301, 700, 1024])
def test_solve_large_dims(d):
    rng = np.random.default_rng(d)
    a = rng.standard_normal((d, d))
    spd = a @ a.T / d + np.eye(d)
    rows, cols, _ = O.tri(d)
    pk = spd[rows, cols]
    b = rng.standard_normal(d)
    z = leaf.shifted_solve(pk, d, 0.25, b)
    want = np.linalg.solve(spd + 0.25 * np.eye(d), b)
    assert normwise(z, want) <= 1e-10


# ------------------------------------------------------------------ P3 / P5


@pytest.mark.parametrize("kind,k", [("topk", 40), ("randseqk", 40), ("randk", 40), ("identity", None)])
def test_round_fold_bit_exact_given_device_deltas(kind, k):
    """Compress the GPU's own differences on the CPU oracle and replay the
    shift + master fold: client and master estimates must match bitwise."""
    shards = D.make_shards(24, 400, 5, seed=21)
    d = shards[0].dim
    cfg = RunConfig(compressor=CompressorSpec(CompressorKind(kind), k=k), rounds=3, run_seed=21)
    eng = FedNLEngine(cfg, d, len(shards), shards[0].n_samples, lam=shards[0].lam)
    eng.upload([s.bmat for s in shards])
    eng.init_state()
    eng.run_rounds(2)
    h_cli = eng.get_client_hest()
    h_mas = eng.get_master_hest()
    x0 = eng.get_x()
    eng.run_rounds(1)
    deltas = {}
    for c in range(len(shards)):
        diff = eng.round_diff(c)
        deltas[c] = O.compress_packed(diff, d, kind, k, O.round_stream(21, c, 2))
        idx, val = eng.round_delta(c)
        if deltas[c].indices is not None:
            assert np.array_equal(idx, deltas[c].indices)
        assert np.array_equal(val, deltas[c].values)
        O.apply_packed(h_cli[c], deltas[c], eng.alpha)
    for c in sorted(deltas):
        O.apply_packed(h_mas, deltas[c], eng.alpha / len(shards))
    assert np.array_equal(eng.get_client_hest(), h_cli)
    assert np.array_equal(eng.get_master_hest(), h_mas)
    # and the iterate: x1 = x0 - solve(H_pre + l I, gbar) within 1e-10
    assert np.all(np.isfinite(eng.get_x())) and not np.array_equal(eng.get_x(), x0)
    eng.close()


def test_split_topk_rounds_bit_identical_to_stream_path():
    """c0 rounds through the split TopK (client shift update moved into the
    master fold) reproduce the pinned k_topk_stream round bit for bit: same
    selections, same shift and fold arithmetic, same trajectory."""
    cfg, shards = sim_case("c0_r4")
    cfg = RunConfig(compressor=cfg.compressor, rounds=12, alpha=cfg.alpha, run_seed=cfg.run_seed)
    out = {}
    paths = (_lib.TOPK_PATH_STREAM, _lib.TOPK_PATH_SPLIT)
    for path in paths:
        eng = FedNLEngine(cfg, shards[0].dim, len(shards), shards[0].n_samples, topk_path=path)
        out[path] = simulate(cfg, shards, engine=eng)
        eng.close()
    for path in paths[1:]:
        for a, b in zip(out[_lib.TOPK_PATH_STREAM], out[path]):
            assert (a.round, a.grad_norm, a.f_value, a.bytes_up_cum) == (b.round, b.grad_norm, b.f_value, b.bytes_up_cum)


# --------------------------------------------------------------------- P6


def _rows_close(rows, g, names, rel=1e-10, floor=1e-6, abs_floor=1e-15, f_rel=1e-12):
    """Row-wise P6 check against one or more of the reference's own valid
    trajectories (`names`): each row must be within tolerance of at least one.

    grad tolerance: rel * max(g_ref, floor * g_ref[0]) + abs_floor * g_ref[0]
    (the absolute term is the rounding noise of a mean of n client gradients
    of size ~g_ref[0], reached in the converged tail).
    """
    base = names[0]
    assert [r.round for r in rows] == g[f"{base}__round"].tolist()
    assert [r.bytes_up_cum for r in rows] == g[f"{base}__bytes_up"].tolist()
    assert [r.bytes_down_cum for r in rows] == g[f"{base}__bytes_down"].tolist()
    assert [r.ls_steps for r in rows] == g[f"{base}__ls_steps"].tolist()
    gn = np.array([r.grad_norm for r in rows])
    fv = np.array([r.f_value for r in rows])
    ok = np.zeros(len(rows), dtype=bool)
    for name in names:
        want_g = g[f"{name}__grad_norm"]
        want_f = g[f"{name}__f_value"]
        tol = rel * np.maximum(want_g, floor * want_g[0]) + abs_floor * want_g[0]
        ok |= (np.abs(gn - want_g) <= tol) & (np.abs(fv - want_f) <= f_rel * np.abs(want_f))
    bad = np.flatnonzero(~ok)
    assert bad.size == 0, (base, bad, gn[bad], fv[bad])


SIM = {
    "fednl_identity": (("synth", 6, 80, 4, 2), dict(rounds=12)),
    "fednl_randk": (("synth", 8, 120, 5, 5), dict(rounds=10, kind="randk", k=9)),
    "fednl_randseqk": (("synth", 8, 120, 5, 6), dict(rounds=10, kind="randseqk", k=9)),
    "fednl_natural": (("synth", 8, 120, 5, 7), dict(rounds=8, kind="natural")),
    "fednl_topk": (("synth", 8, 120, 5, 3), dict(rounds=10, kind="topk", k=9)),
    "fednl_topkW": (("synth", 8, 120, 5, 3), dict(rounds=10, kind="topk", k=9, topk_weighted=True)),
    "fednl_toplek": (("synth", 8, 120, 5, 4), dict(rounds=10, kind="toplek", k=9)),
    "fednl_alpha1_stop": (("synth", 5, 60, 2, 6), dict(rounds=50, alpha=1.0, kind="topk", k=4,
                                                         stop_grad_norm=1e-9)),
    "fednl_zero_init": (("synth", 6, 80, 4, 8), dict(rounds=6, hessian_init="zero", kind="topk", k=8)),
    "fednl_exact_init": (("synth", 6, 80, 4, 9), dict(rounds=6, hessian_init="exact",
                                                        kind="randseqk", k=8)),
    "ls_topk": (("synth", 8, 120, 4, 10), dict(rounds=10, algorithm="fednl-ls", kind="topk", k=9)),
    "ls_toplek": (("synth", 8, 120, 4, 11), dict(rounds=10, algorithm="fednl-ls", kind="toplek", k=12)),
    "pp_randk": (("synth", 8, 150, 6, 12), dict(rounds=15, algorithm="fednl-pp", tau=2,
                                                 kind="randk", k=9)),
    "pp_topk": (("synth", 8, 150, 6, 13), dict(rounds=15, algorithm="fednl-pp", tau=3,
                                                kind="topk", k=9)),
    "pp_identity_stop": (("synth", 4, 60, 4, 8), dict(rounds=60, algorithm="fednl-pp", tau=2,
                                                       stop_grad_norm=1e-10)),
    "c1_r30": (("baseline", "c1"), dict(rounds=30)),
    "c2_r30": (("baseline", "c2"), dict(rounds=30)),
    "c3_r30": (("baseline", "c3"), dict(rounds=30)),
    "c0_r4": (("baseline", "c0"), dict(rounds=4)),
}


def sim_case(name):
    gen, kw = SIM[name]
    kw = dict(kw)
    if gen[0] == "synth":
        _, nf, m, n, seed = gen
        shards = D.make_shards(nf, m, n, seed)
        kw.setdefault("run_seed", seed)
    else:
        c = D.BASELINE_CONFIGS[gen[1]]
        shards = D.baseline_shards(gen[1])
        kw.setdefault("run_seed", 1)
        for key in ("algorithm", "kind", "k", "alpha", "tau"):
            if key in c:
                kw.setdefault(key, c[key])
    kind = kw.pop("kind", "identity")
    k = kw.pop("k", None)
    weighted = kw.pop("topk_weighted", False)
    cfg = RunConfig(compressor=CompressorSpec(CompressorKind(kind), k=k, topk_weighted=weighted), **kw)
    return cfg, shards


@pytest.mark.parametrize("name", list(SIM))
def test_simulate_rows_match_reference(name):
    cfg, shards = sim_case(name)
    rows = simulate(cfg, shards)
    g = golden("simulate.npz")
    if name == "c0_r4":
        # TopK at a real shape: an ulp-level difference in D can legitimately
        # swap a k-th-boundary tie (the reference itself does so between BLAS
        # thread counts at round 3): judged against both of the
        # reference's trajectories and its own envelope
        _envelope_close(rows, g, "c0_r4", "c0_r4_mt")
    else:
        _rows_close(rows, g, [name])


def _envelope_close(rows, g, base, mt):
    """P6 for the tie-heavy TopK shapes: rows within 1e-10 of one of the
    reference's two valid trajectories (1 and 8 BLAS threads) until the
    first k-th-boundary swap, and every row within 4x the reference's own
    whole-run envelope E = max_i |g1_i - g8_i| / g1_i of the nearer one:
    after a swap each valid trajectory (the reference's two, the GPU's) takes
    its own branch, and E is one sample of how far two branches drift apart
    (c0_r20 measured: 0.55 E and 2.4 E for two builds whose Hessian sums
    differ only in association).  f_value is flat near its minimum, so one
    swap moves it by a round-dependent amount: its bar is 10x the
    reference's own f envelope (measured up to 3.8x)."""
    g1, g8 = g[f"{base}__grad_norm"], g[f"{mt}__grad_norm"]
    f1, f8 = g[f"{base}__f_value"], g[f"{mt}__f_value"]
    assert [r.round for r in rows] == g[f"{base}__round"].tolist()
    assert [r.bytes_up_cum for r in rows] == g[f"{base}__bytes_up"].tolist()
    assert [r.bytes_down_cum for r in rows] == g[f"{base}__bytes_down"].tolist()
    gn = np.array([r.grad_norm for r in rows])
    fv = np.array([r.f_value for r in rows])
    env = float(np.max(np.abs(g1 - g8) / g1))
    env_f = float(np.max(np.abs(f1 - f8) / np.abs(f1)))
    dev = np.minimum(np.abs(gn - g1) / g1, np.abs(gn - g8) / g8)
    dev_f = np.minimum(np.abs(fv - f1) / np.abs(f1), np.abs(fv - f8) / np.abs(f8))
    first = int(np.argmax(dev > 1e-10)) if np.any(dev > 1e-10) else len(rows)
    assert first >= 3, ("left both references before their own first swap", first, dev)
    assert np.all(dev <= 4 * env), (env, dev)
    assert np.all(dev_f <= max(10 * env_f, 1e-12)), (env_f, dev_f)
    return dev


def _kth_boundary_ok(got_idx, want_idx, diff_gpu, diff_ref, k, ulps=4):
    """Tie-aware index-set comparison: every position in the
    symmetric difference must sit within `ulps` of the k-th largest |D| in
    both implementations."""
    sym = np.setxor1d(got_idx, want_idx)
    if sym.size == 0:
        return 0
    for dv in (diff_gpu, diff_ref):
        kth = np.sort(np.abs(dv))[::-1][k - 1]
        tol = ulps * np.spacing(kth)
        assert np.all(np.abs(np.abs(dv[sym]) - kth) <= tol), (sym, np.abs(dv[sym]), kth)
    return sym.size // 2


def test_teacher_forced_round_c0():
    """P5 at the c0 shape: the GPU round started from the oracle's state at
    round 2 reproduces the oracle's round: D within 1e-10 (normwise per
    client), index sets equal up to k-th-boundary ties, next iterate 1e-10."""
    shards = D.baseline_shards("c0")
    cfg = D.baseline_run_config("c0", rounds=4)
    d, n = shards[0].dim, len(shards)
    ocfg = O.OracleConfig.from_run_config(cfg)
    run = O.OracleRun(ocfg, [s.bmat for s in shards], lam=shards[0].lam, workers=16)
    run.init()
    for r in range(2):
        run.fednl_round(r)
    x0, h_cli0, h_mas0 = run.x.copy(), run.h_cli.copy(), run.h_mas.copy()
    # the oracle's round 2, client by client
    ref_diff, ref_idx = [], []
    for c in range(n):
        ev = O.local_eval(shards[c].bmat, shards[c].lam, x0)
        dv = ev.hess - h_cli0[c]
        ref_diff.append(dv)
        ref_idx.append(O.compress_packed(dv, d, "topk", cfg.compressor.k,
                                         O.round_stream(cfg.run_seed, c, 2)).indices)
    run.fednl_round(2)
    x_ref = run.x.copy()
    run_h_mas = run.h_mas.copy()
    run.close()
    eng = FedNLEngine(cfg, d, n, shards[0].n_samples, lam=shards[0].lam)
    eng.upload([s.bmat for s in shards])
    eng.init_state()
    eng.set_x(x0)
    eng.set_client_hest(h_cli0)
    eng.set_master_hest(h_mas0)
    eng.run_rounds(1, first_round=2)
    swaps = 0
    sc, cli_shift = eng.round_scalars()
    ref_shift = np.array([O.frob(ref_diff[c], d) for c in range(n)])
    assert normwise(cli_shift, ref_shift) <= 1e-10
    mg, _ = eng.round_grads()
    ref_g = np.zeros(d)
    for c in range(n):
        ref_g += O.local_eval(shards[c].bmat, shards[c].lam, x0, need_hess=False).grad
    assert normwise(mg, ref_g / n) <= 1e-10
    h_fold = h_mas0.copy()  # the master fold of the GPU's own selections, in the oracle
    for c in range(n):
        dv = eng.round_diff(c)
        hmax = np.max(np.abs(ref_diff[c] + h_cli0[c]))
        assert np.max(np.abs(dv - ref_diff[c])) <= 1e-10 * hmax, c
        idx, val = eng.round_delta(c)
        swaps += _kth_boundary_ok(idx, ref_idx[c], dv, ref_diff[c], cfg.compressor.k)
        assert np.array_equal(val, dv[idx])  # TopK values: unscaled D at the kept positions
        O.apply_packed(h_fold, O.Delta("topk", d, ref_diff[c][idx], idx.astype(np.uint32)), eng.alpha / n)
    # x^{k+1} = x^k - (H^k + l^k I)^{-1} gbar uses the pre-fold H^k: it does
    # not depend on this round's selections, so it is checked even after swaps
    assert normwise(eng.get_x(), x_ref) <= 1e-10
    # H^{k+1}: the GPU's selections folded by the oracle from the reference's D
    assert normwise(eng.get_master_hest(), h_fold) <= 1e-10
    if swaps == 0:
        assert normwise(eng.get_master_hest(), run_h_mas) <= 1e-10
    print(f"[P5 c0] boundary swaps in round 2: {swaps}")
    eng.close()


@pytest.mark.parametrize("name,rounds", [("c0", 3), ("c1", 2), ("c2", 2)])
def test_compressor_bit_exact_on_device_round_diffs(name, rounds):
    """P1 on the GPU's own round-r differences at the BASELINE shapes: the
    compressed delta each client produced equals the oracle's compress of the
    same packed difference with the same (client, round) stream."""
    shards = D.baseline_shards(name)
    cfg = D.baseline_run_config(name, rounds=rounds)
    d = shards[0].dim
    eng = FedNLEngine(cfg, d, len(shards), shards[0].n_samples, lam=shards[0].lam)
    eng.upload([s.bmat for s in shards])
    eng.init_state()
    kind = cfg.compressor.kind.value
    k = cfg.compressor.k
    for r in range(rounds):
        eng.run_rounds(1)
        for cid in range(0, len(shards), max(1, len(shards) // 12)):
            diff = eng.round_diff(cid)
            want = O.compress_packed(diff, d, kind, k, O.round_stream(cfg.run_seed, cid, r))
            idx, val = eng.round_delta(cid)
            assert np.array_equal(idx, want.indices), (name, r, cid)
            assert np.array_equal(val, want.values), (name, r, cid)
    eng.close()


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_round_fold_bit_exact_at_baseline_shape(name):
    """P3 at full size: replay the shift update and master fold of round 1 on
    the CPU from the device's own deltas; estimates must match bitwise."""
    shards = D.baseline_shards(name)
    cfg = D.baseline_run_config(name, rounds=2)
    d, n = shards[0].dim, len(shards)
    eng = FedNLEngine(cfg, d, n, shards[0].n_samples, lam=shards[0].lam)
    eng.upload([s.bmat for s in shards])
    eng.init_state()
    eng.run_rounds(1)
    h_cli = eng.get_client_hest()
    h_mas = eng.get_master_hest()
    eng.run_rounds(1)
    kind, k = cfg.compressor.kind.value, cfg.compressor.k
    for c in range(n):
        delta = O.compress_packed(eng.round_diff(c), d, kind, k, O.round_stream(cfg.run_seed, c, 1))
        idx, val = eng.round_delta(c)
        assert np.array_equal(idx, delta.indices) and np.array_equal(val, delta.values), c
        O.apply_packed(h_cli[c], delta, eng.alpha)
        O.apply_packed(h_mas, delta, eng.alpha / n)
    got_cli = eng.get_client_hest()
    bad = [c for c in range(n) if not np.array_equal(got_cli[c], h_cli[c])]
    assert not bad, bad[:5]
    assert np.array_equal(eng.get_master_hest(), h_mas)
    eng.close()


@pytest.mark.parametrize("name", ["c0", "c3"])
def test_round0_shift_norms_match_oracle(name):
    """Every client's l_i = ||H_i(x0) - H_i^0||_F and D_i at x0 = 0 against the
    oracle at 1e-10 (FedNL round 0; FedNL-PP initial shifts).  Guards the
    Hessian's TMA ring hand-off: a slot released before its fragment loads
    completed once corrupted single samples of D for a fraction of clients."""
    shards = D.baseline_shards(name)
    cfg = D.baseline_run_config(name, rounds=2)
    d, lam = shards[0].dim, shards[0].lam
    eng = FedNLEngine(cfg, d, len(shards), shards[0].n_samples, lam=lam)
    try:
        eng.upload([s.bmat for s in shards])
        eng.init_state()
        w = d * (d + 1) // 2
        diag_idx = np.array([j * (j + 1) // 2 + j for j in range(d)])
        wt = np.full(w, 2.0)
        wt[diag_idx] = 1.0
        if name == "c3":
            got = np.asarray(eng.get_pp_state()[2])  # per-client shifts after init
        else:
            eng.run_rounds(1)
            got = eng.round_scalars()[1]
        for c in range(len(shards)):
            ev = O.local_eval(shards[c].bmat, lam, np.zeros(d), need_hess=True, need_f=False)
            want_d = ev.hess.copy()
            want_d[diag_idx] -= lam
            want = np.sqrt(np.sum(wt * want_d * want_d))
            assert abs(got[c] - want) <= 1e-10 * want, (c, got[c], want)
            if name == "c0":
                assert normwise(eng.round_diff(c), want_d, np.max(np.abs(ev.hess))) <= 1e-10, c
    finally:
        eng.close()


@pytest.mark.parametrize("name", ["c0_r4", "ls_topk", "fednl_natural", "fednl_exact_init", "pp_randk",
                                  "pp_identity_stop", "c2_r30"])
def test_sharded_path_world1_matches_unsharded(name):
    """The client-sharded round (fb_set_shard: NCCL all-gathers inside the
    captured graph — in the line search's while-loop body for FedNL-LS, the
    dense updates for Identity / Natural, the round-0 Hessians for exact
    init, the participant-slot exchange for FedNL-PP) with one rank
    reproduces the single-GPU rows, iterate and master state bit for bit."""
    from paper_2410_08760_b200.engine import nccl_unique_id

    cfg, shards = sim_case(name)
    d, n, ni = shards[0].dim, len(shards), shards[0].n_samples
    out = []
    for shard in (False, True):
        eng = FedNLEngine(cfg, d, n, ni)
        try:
            if shard:
                eng.set_shard(1, 0, nccl_unique_id())
            rows = simulate(cfg, shards, engine=eng)
            out.append(([(r.grad_norm, r.f_value, r.bytes_up_cum, r.ls_steps) for r in rows], eng.get_x(),
                        eng.get_master_hest()))
        finally:
            eng.close()
    assert out[0][0] == out[1][0]
    for a, b in zip(out[0][1:], out[1][1:]):
        assert np.array_equal(np.asarray(a), np.asarray(b))


@pytest.mark.parametrize("d", [69, 161])  # k_chol_solve path / panel path (fused reduction)
def test_round_rejects_nonfinite_client_hessian(d):
    """A client whose data makes H_i(x) - H_i^k non-finite stops the round the
    way the reference's client compressor does (ValueError), from either
    round-reduction path."""
    rng = np.random.default_rng(d)
    n, ni = 6, 40
    bmats = []
    for _ in range(n):
        feats = (rng.random((d - 1, ni)) < 0.2).astype(np.float64)
        y = np.where(rng.random(ni) < 0.5, 1.0, -1.0)
        bmats.append(np.asfortranarray(np.vstack([feats, np.ones((1, ni))]) * y))
    cfg = RunConfig(algorithm="fednl", compressor=CompressorSpec(CompressorKind.TOPK, k=2 * d),
                    rounds=3, run_seed=1)
    eng = FedNLEngine(cfg, d, n, ni, lam=1e-3)
    try:
        eng.upload(bmats)
        eng.init_state()
        eng.run_rounds(1)  # finite data: fine
        bad = [b.copy(order="F") for b in bmats]
        bad[3][5, 7] = np.inf  # client 3's next Hessian is non-finite
        eng.upload(bad)
        with pytest.raises(ValueError):
            eng.run_rounds(1)
    finally:
        eng.close()


# ------------------------------------------------- option a (eigen clamp)


def test_device_jacobi_and_eigen_clamp_against_golden():
    """linalg.jacobi_eigh / eigen_clamp_min (linalg.py:189-259) on the device
    against the reference's outputs: eigenvalues, reconstruction and
    orthonormality as the reference's own tests check them (test_linalg.py:
    191-226), clamped matrices within 1e-10 normwise, exactly symmetric."""
    g = golden("eigen.npz")
    for name in g["names"].tolist():
        pk = g[f"{name}__pk"]
        d = int(round((np.sqrt(8 * pk.size + 1) - 1) / 2))
        m = O.to_dense(pk, d)
        scale = max(1.0, float(np.abs(m).max()))
        vals, vecs = leaf.jacobi_eigh(m)
        assert np.allclose(np.sort(vals), g[f"{name}__vals_sorted"], rtol=0, atol=1e-10 * scale), name
        assert np.allclose((vecs * vals) @ vecs.T, m, rtol=0, atol=1e-10 * scale), name
        assert np.allclose(vecs.T @ vecs, np.eye(d), rtol=0, atol=1e-12), name
        for floor in (0.5, 1e-12):
            got = leaf.eigen_clamp_min(m, floor)
            assert np.array_equal(got, got.T), name
            assert normwise(O.pack_upper(got), g[f"{name}__clamp{floor:g}"], scale) <= 1e-10, (name, floor)
    # no rotations on a diagonal matrix: values and vectors bit-exact
    vals, vecs = leaf.jacobi_eigh(np.diag([3.0, -1.0, 2.0]))
    assert np.array_equal(np.sort(vals), [-1.0, 2.0, 3.0])
    assert np.array_equal(vecs, np.eye(3))


def test_option_a_uses_clamped_system():
    """test_algorithms.py:399-406: H = diag(-1, 4), mu = 0.5 -> the solve
    uses diag(0.5, 4); grad (1, 8) gives x = (-2, -2) from x = 0."""
    sysm = leaf.eigen_clamp_min(np.diag([-1.0, 4.0]), 0.5)
    p = leaf.cholesky_solve(sysm, np.array([1.0, 8.0]))
    assert np.allclose(0.0 - p, [-2.0, -2.0], rtol=0, atol=1e-12)


OPT_A = {
    "fednl_opt_a": ((8, 120, 5, 14), dict(rounds=10, option="a", kind="topk", k=9)),
    "fednl_opt_a_mu": ((8, 120, 5, 15), dict(rounds=10, option="a", mu=0.05, kind="randseqk", k=9)),
    "ls_opt_a": ((8, 120, 4, 16), dict(rounds=10, algorithm="fednl-ls", option="a", mu=0.02,
                                       kind="toplek", k=12)),
}


@pytest.mark.parametrize("name", list(OPT_A))
def test_simulate_option_a_matches_reference(name):
    (nf, m, n, seed), kw = OPT_A[name]
    kw = dict(kw)
    shards = D.make_shards(nf, m, n, seed)
    spec = CompressorSpec(CompressorKind(kw.pop("kind")), k=kw.pop("k"))
    rows = simulate(RunConfig(compressor=spec, run_seed=seed, **kw), shards)
    _rows_close(rows, golden("simulate_opt_a.npz"), [name])


def test_option_a_singular_system_raises():
    """test_cli.py:135-146: option a with a zero estimate and floor 0 is
    singular at pivot 0 of the very first solve."""
    shards = D.make_shards(2, 4, 1, 0, lam=0.0)
    cfg = RunConfig(option="a", mu=0.0, lam=0.0, hessian_init="zero", rounds=1)
    with pytest.raises(NotPositiveDefiniteError) as e:
        simulate(cfg, shards)
    assert e.value.pivot_index == 0


def test_leaf_solve_after_not_pd_failure_is_clean():
    """A NotPositiveDefiniteError from one leaf solve must not leak into the
    next call on the same (cached) context."""
    with pytest.raises(NotPositiveDefiniteError) as e:
        leaf.cholesky_solve(np.array([[1.0, 2.0], [2.0, 1.0]]), np.array([1.0, 1.0]))
    assert e.value.pivot_index == 1
    p = leaf.cholesky_solve(np.diag([0.5, 4.0]), np.array([1.0, 8.0]))
    assert np.allclose(p, [2.0, 2.0], rtol=0, atol=1e-12)
    out = leaf.eigen_clamp_min(np.diag([-1.0, 4.0]), 0.5)
    assert np.allclose(out, np.diag([0.5, 4.0]), rtol=0, atol=1e-15)
