"""Pin the CPU oracle (oracle/fednl_oracle.py) to the reference's own outputs.

The golden vectors in tests/golden/ were produced by running the reference
(oracle/make_golden.py).  Integer / index / PRNG outputs and compressor
outputs on fixed inputs must match bit for bit; BLAS-evaluated floats match
bit for bit on the build host with OPENBLAS_NUM_THREADS=1 and within 1e-12
elsewhere.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from oracle import fednl_oracle as O
from paper_2410_08760_b200 import data as D
from paper_2410_08760_b200 import rng as R

SEED0_PUBLISHED = [  # the widely published SplitMix64 seed-0 vector (test_rng.py:22-28)
    0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F,
    0xF88BB8A8724C81EC, 0x1B39896A51A8749B,
]


# ------------------------------------------------------------------ PRNG (P0)


def test_seed0_stream_matches_published_and_golden():
    g = golden("rng.npz")
    assert [int(v) for v in g["seed0_stream"]] == SEED0_PUBLISHED
    p = O.SplitMix64(0)
    assert [p.next_u64() for _ in range(5)] == SEED0_PUBLISHED
    q = R.Prg(0)
    assert [q.next_u64() for _ in range(5)] == SEED0_PUBLISHED


def test_streams_blocks_and_f64():
    g = golden("rng.npz")
    for a, s in enumerate(g["stream_seeds"].tolist()):
        assert np.array_equal(O.SplitMix64(s).u64_block(64), g["streams"][a])
        assert np.array_equal(R.Prg(s).u64_block(64), g["streams"][a])
        p = O.SplitMix64(s)
        assert [p.next_u64() for _ in range(64)] == g["streams"][a].tolist()
        assert np.array_equal(O.SplitMix64(s).f64_block(64), g["f64_streams"][a])
        p = O.SplitMix64(s)
        assert [p.next_f64() for _ in range(64)] == g["f64_streams"][a].tolist()


def test_randrange_and_draw_consumption():
    g = golden("rng.npz")
    for a, s in enumerate(g["stream_seeds"].tolist()):
        for b, bd in enumerate(g["rr_bounds"].tolist()):
            for impl in (O.SplitMix64, R.Prg):
                p = impl(s)
                assert [p.randrange(bd) for _ in range(8)] == g["randrange"][a, b].tolist()
                assert p.next_u64() == int(g["randrange_next"][a, b])


def test_partial_shuffles_and_master_subsets():
    g = golden("rng.npz")
    for key in ("randk_c3", "pp_c3", "small", "full"):
        n, k, s = (int(v) for v in g[f"pshuffle_{key}_args"])
        assert np.array_equal(O.SplitMix64(s).partial_shuffle_prefix(n, k), g[f"pshuffle_{key}"])
        assert np.array_equal(R.Prg(s).partial_shuffle_prefix(n, k), g[f"pshuffle_{key}"])
    mp = O.named_stream(1, O.TAG_MASTER)
    subs = np.stack([np.sort(mp.partial_shuffle_prefix(142, 12)) for _ in range(20)])
    assert np.array_equal(subs, g["pp_subsets_c3"])


def test_round_seed_grid_and_tags():
    g = golden("rng.npz")
    assert g["tags"].tolist() == [O.TAG_SHUFFLE, O.TAG_SYNTH, O.TAG_MASTER]
    for a, rs in enumerate([0, 1, 123, (1 << 64) - 1]):
        for c in range(6):
            for r in range(6):
                want = int(g["round_seed_grid"][a, c, r])
                assert O.round_seed(rs, c * 1000 + c, r * 77 + r) == want
                assert R.derive_round_seed(rs, c * 1000 + c, r * 77 + r) == want


def test_round_seed_range_checks():
    with pytest.raises(ValueError):
        O.round_seed(0, 1 << 32, 0)
    with pytest.raises(ValueError):
        R.derive_round_seed(0, 0, -1)


# ---------------------------------------------------------- compressors (P1)


def _compress_tags(g):
    for name in g["case_names"].tolist():
        pk = g[f"{name}__input"]
        d = int(g[f"{name}__d"])
        for key in g.files:
            if key.startswith(name + "__") and key.endswith("__val"):
                yield name, d, pk, key[len(name) + 2:-5]


def test_compressors_bit_exact_against_reference_outputs():
    g = golden("compress.npz")
    n_checked = 0
    for name, d, pk, tag in _compress_tags(g):
        parts = tag.split("__")
        kind = parts[0]
        weighted = kind.endswith("W")
        kind = kind.rstrip("W")
        if kind in ("identity", "natural"):
            k, seed = None, int(parts[1][1:])
        else:
            k, seed = int(parts[1][1:]), int(parts[2][1:])
        prg = O.SplitMix64(seed)
        delta = O.compress_packed(pk, d, kind, k, prg, topk_weighted=weighted)
        base = f"{name}__{tag}"
        assert np.array_equal(delta.values, g[base + "__val"]), base
        if base + "__idx" in g.files:
            assert np.array_equal(delta.indices, g[base + "__idx"]), base
        assert prg.next_u64() == int(g[base + "__next"]), base
        n_checked += 1
    assert n_checked > 300


def test_topk_round0_full_c0_shape():
    """The tie-heavy round-0 TopK sets at the full c0 shape (x = 0)."""
    g = golden("topk_c0_round0.npz")
    shards = D.baseline_shards("c0")
    d = shards[0].dim
    for cid in (0, 1, 77, 141):
        ev = O.local_eval(shards[cid].bmat, 1e-3, np.zeros(d))
        diff = ev.hess.copy()
        diff[O.diag_positions(d)] = diff[O.diag_positions(d)] - 1e-3
        delta = O.compress_packed(diff, d, "topk", 2408, O.round_stream(1, cid, 0))
        assert np.array_equal(delta.indices, g[f"cid{cid}__idx"])
        assert np.array_equal(delta.values, g[f"cid{cid}__val"])


def test_numpy_pairwise_sum_restatement():
    rng = np.random.default_rng(3)
    for n in (1, 7, 8, 9, 127, 128, 129, 1000, 2415, 4097):
        a = np.abs(rng.standard_normal(n)) * 10.0 ** rng.integers(-8, 8, n)
        assert O.numpy_pairwise_sum(a) == float(np.sum(a))


def test_toplek_plan_hand_cases():
    assert O.toplek_plan(np.array([4.0, 1.0, 1.0]), 1)[:2] == (0, 1)
    assert abs(O.toplek_plan(np.array([4.0, 1.0, 1.0]), 1)[2] - 0.5) < 1e-15
    assert O.toplek_plan(np.array([2.0, 2.0, 2.0]), 1) == (1, 1, 1.0)
    with pytest.raises(ValueError):
        O.toplek_plan(np.zeros(3), 1)


def test_zero_and_nonfinite_inputs():
    for kind in ("identity", "topk", "toplek", "randk", "randseqk", "natural"):
        prg = O.SplitMix64(9)
        delta = O.compress_packed(np.zeros(10), 4, kind, 2, prg)
        assert delta.count == 0 and O.wire_bytes(delta, True) == 0
        assert prg.next_u64() == O.SplitMix64(9).next_u64()
    bad = np.zeros(3)
    bad[1] = np.nan
    with pytest.raises(ValueError):
        O.compress_packed(bad, 2, "identity", None, O.SplitMix64(0))


# --------------------------------------------------------------- oracle (P2)


def test_local_oracle_against_reference_values():
    g = golden("oracle.npz")
    lam = float(g["lam"])
    for ci in range(3):
        b = g[f"bmat{ci}"]
        for xi, x in enumerate(g["xs"]):
            ev = O.local_eval(np.asfortranarray(b), lam, x)
            for got, key in ((ev.f, "f"), (ev.grad, "grad"), (ev.hess, "hess")):
                want = g[f"{key}_{ci}_{xi}"]
                scale = max(1.0, float(np.max(np.abs(want))))
                assert np.max(np.abs(np.asarray(got) - want)) <= 1e-12 * scale


# ----------------------------------------------------------------- solve (P4)


def test_cholesky_solves_and_pivot_errors():
    g = golden("linalg.npz")
    for d in (1, 2, 10, 50, 301):
        x = O.shifted_solve(g[f"spd{d}"], d, 0.0, g[f"rhs{d}"])
        want = g[f"sol{d}"]
        assert np.max(np.abs(x - want)) <= 1e-12 * max(1.0, np.max(np.abs(want)))
    for key in ("npd", "npd2"):
        pk = g[f"{key}_pk"]
        d = int((np.sqrt(8 * len(pk) + 1) - 1) / 2)
        with pytest.raises(O.NotPD) as exc:
            O.shifted_solve(pk, d, 0.0, np.ones(d))
        assert exc.value.pivot_index == int(g[f"{key}_pivot"][0])
        assert exc.value.pivot_value == pytest.approx(float(g[f"{key}_pivot"][1]), rel=1e-12)


# ------------------------------------------------------------- data builders


def test_shard_builders_match_reference_bytes():
    g = golden("data.npz")
    for name in ("c0", "c1", "c2"):
        sh = D.baseline_shards(name)
        assert np.array_equal(np.stack([s.bmat.sum(axis=0) for s in sh[:4]]), g[f"{name}__colsum"])
        assert np.array_equal(np.stack([s.bmat.sum(axis=1) for s in sh]), g[f"{name}__rowsum"])
        assert np.array_equal(np.stack([s.bmat[:, 0] for s in sh]), g[f"{name}__first_col"])
        assert all(s.bmat.flags.f_contiguous for s in sh)
    sh = D.make_shards(6, 90, 3, seed=5, lam=0.01)
    assert np.array_equal(np.stack([s.bmat for s in sh]), g["synth_6_90_3_5"])


# ------------------------------------------------------- whole runs (P5/P6)

SIM_CASES = {
    "fednl_identity": (("synth", 6, 80, 4, 2), dict(rounds=12)),
    "fednl_topk": (("synth", 8, 120, 5, 3), dict(rounds=10, kind="topk", k=9)),
    "fednl_topkW": (("synth", 8, 120, 5, 3), dict(rounds=10, kind="topk", k=9, topk_weighted=True)),
    "fednl_toplek": (("synth", 8, 120, 5, 4), dict(rounds=10, kind="toplek", k=9)),
    "fednl_randk": (("synth", 8, 120, 5, 5), dict(rounds=10, kind="randk", k=9)),
    "fednl_randseqk": (("synth", 8, 120, 5, 6), dict(rounds=10, kind="randseqk", k=9)),
    "fednl_natural": (("synth", 8, 120, 5, 7), dict(rounds=8, kind="natural")),
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


def sim_inputs(name):
    gen, kw = SIM_CASES[name]
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
    return O.OracleConfig(**kw), shards


@pytest.mark.parametrize("name", list(SIM_CASES))
def test_oracle_simulate_matches_reference_rows(name):
    cfg, shards = sim_inputs(name)
    rows = O.simulate(cfg, [s.bmat for s in shards], lam=shards[0].lam)
    g = golden("simulate.npz")
    assert [r.round for r in rows] == g[f"{name}__round"].tolist()
    assert [r.bytes_up_cum for r in rows] == g[f"{name}__bytes_up"].tolist()
    assert [r.bytes_down_cum for r in rows] == g[f"{name}__bytes_down"].tolist()
    assert [r.ls_steps for r in rows] == g[f"{name}__ls_steps"].tolist()
    # same BLAS + same order => bitwise on the build host; allow rounding-level
    # slack elsewhere
    gn = np.array([r.grad_norm for r in rows])
    fv = np.array([r.f_value for r in rows])
    want_g, want_f = g[f"{name}__grad_norm"], g[f"{name}__f_value"]
    assert np.all(np.abs(gn - want_g) <= 1e-9 * np.maximum(want_g, 1e-6 * want_g[0]))
    assert np.all(np.abs(fv - want_f) <= 1e-12 * np.abs(want_f))


def test_worker_count_invariance():
    cfg, shards = sim_inputs("fednl_topk")
    a = O.simulate(cfg, [s.bmat for s in shards], lam=shards[0].lam, workers=1)
    b = O.simulate(cfg, [s.bmat for s in shards], lam=shards[0].lam, workers=4)
    for r1, r2 in zip(a, b):
        assert (r1.grad_norm, r1.f_value, r1.bytes_up_cum) == (r2.grad_norm, r2.f_value, r2.bytes_up_cum)


# ------------------------------------------------- option a (eigen clamp)


def test_jacobi_and_eigen_clamp_match_reference():
    """jacobi_eigh / eigen_clamp_min restated (linalg.py:189-259): the same
    cyclic Jacobi in the same order, so the reference's outputs come back to
    rounding of the final BLAS product."""
    g = golden("eigen.npz")
    for name in g["names"].tolist():
        pk = g[f"{name}__pk"]
        d = int(round((np.sqrt(8 * pk.size + 1) - 1) / 2))
        m = O.to_dense(pk, d)
        vals, vecs = O.jacobi_eigh(m)
        scale = max(1.0, float(np.abs(m).max()))
        assert np.allclose(np.sort(vals), g[f"{name}__vals_sorted"], rtol=0, atol=1e-12 * scale), name
        assert np.allclose(vecs.T @ vecs, np.eye(d), rtol=0, atol=1e-12), name
        for floor in (0.5, 1e-12):
            got = O.pack_upper(O.eigen_clamp_min(m, floor))
            assert np.allclose(got, g[f"{name}__clamp{floor:g}"], rtol=0, atol=1e-12 * scale), (name, floor)


OPT_A = {
    "fednl_opt_a": (("synth", 8, 120, 5, 14), dict(rounds=10, option="a", kind="topk", k=9)),
    "fednl_opt_a_mu": (("synth", 8, 120, 5, 15), dict(rounds=10, option="a", mu=0.05,
                                                       kind="randseqk", k=9)),
    "ls_opt_a": (("synth", 8, 120, 4, 16), dict(rounds=10, algorithm="fednl-ls", option="a",
                                                 mu=0.02, kind="toplek", k=12)),
}


@pytest.mark.parametrize("name", list(OPT_A))
def test_oracle_option_a_matches_reference_rows(name):
    (_, nf, m, n, seed), kw = OPT_A[name]
    shards = D.make_shards(nf, m, n, seed)
    cfg = O.OracleConfig(run_seed=seed, **kw)
    rows = O.simulate(cfg, [s.bmat for s in shards], lam=shards[0].lam)
    g = golden("simulate_opt_a.npz")
    assert [r.round for r in rows] == g[f"{name}__round"].tolist()
    assert [r.bytes_up_cum for r in rows] == g[f"{name}__bytes_up"].tolist()
    assert [r.ls_steps for r in rows] == g[f"{name}__ls_steps"].tolist()
    gn = np.array([r.grad_norm for r in rows])
    want_g = g[f"{name}__grad_norm"]
    assert np.all(np.abs(gn - want_g) <= 1e-9 * np.maximum(want_g, 1e-6 * want_g[0]))


# ------------------------------------------------- round-2 cases (simulate_r2)

from cases_r2 import LS_FAIL, SIM_R2, case_r2  # noqa: E402


@pytest.mark.parametrize("name", [n for n in SIM_R2 if n != "c0_r20"])
def test_oracle_round2_cases_match_reference_rows(name):
    """Deep line searches, ragged shards with per-shard lambda: the oracle
    restatement reproduces the reference's rows (bitwise on one BLAS thread)."""
    kw, shards = case_r2(name)
    cfg = O.OracleConfig(**kw)
    rows = O.simulate(cfg, [s.bmat for s in shards], lam=[s.lam for s in shards])
    g = golden("simulate_r2.npz")
    assert [r.round for r in rows] == g[f"{name}__round"].tolist()
    assert [r.bytes_up_cum for r in rows] == g[f"{name}__bytes_up"].tolist()
    assert [r.bytes_down_cum for r in rows] == g[f"{name}__bytes_down"].tolist()
    assert [r.ls_steps for r in rows] == g[f"{name}__ls_steps"].tolist()
    assert np.array_equal([r.grad_norm for r in rows], g[f"{name}__grad_norm"])
    assert np.array_equal([r.f_value for r in rows], g[f"{name}__f_value"])


def test_oracle_line_search_failure_matches_reference():
    kw, shards = case_r2(LS_FAIL["base"])
    kw.update(ls_c=LS_FAIL["ls_c"], ls_gamma=LS_FAIL["ls_gamma"], rounds=LS_FAIL["rounds"])
    g = golden("simulate_r2.npz")
    with pytest.raises(O.LineSearchFailed) as exc:
        O.simulate(O.OracleConfig(**kw), [s.bmat for s in shards], lam=shards[0].lam)
    assert exc.value.round == int(g["ls_fail__round"])


def test_large_w_toplek_and_randk_against_reference():
    """TopLEK at w = 45,451 (c0 round-0 differences: heavy ties) and RandK
    with k > 6000: the restatement matches the reference bit for bit."""
    g = golden("compress_r2.npz")
    d = int(g["d"])
    n_checked = 0
    for name in g["names"].tolist():
        pk = g[f"{name}__input"]
        for key in g.files:
            if key.startswith(name + "__") and key.endswith("__val"):
                tag = key[len(name) + 2:-5]
                kind, k, seed = tag.split("__")
                prg = O.SplitMix64(int(seed[1:]))
                delta = O.compress_packed(pk, d, kind, int(k[1:]), prg)
                base = f"{name}__{tag}"
                assert np.array_equal(delta.values, g[base + "__val"]), base
                assert np.array_equal(delta.indices, g[base + "__idx"]), base
                assert prg.next_u64() == int(g[base + "__next"]), base
                n_checked += 1
    assert n_checked == 40


def test_csv_and_canonical_config_match_reference_text(tmp_path):
    """write_csv (with and without the '# config:' line) and canonical_config
    produce the reference's bytes (runtime.py:69-113, transport.py:205-232);
    read_csv round-trips every float exactly."""
    import io

    from paper_2410_08760_b200 import CompressorKind, CompressorSpec, RunConfig
    from paper_2410_08760_b200.runtime import MetricsRow, canonical_config, read_csv, write_csv

    g = golden("csv.npz")
    rows = [MetricsRow(0, 0.0, 0.24282060357349974, 0.6931471805599453, 0, 42784, 0),
            MetricsRow(1, 0.012345678901234568, 1e-300, -0.0, 31312, 85568, 3),
            MetricsRow(2, 1.5, 5e-324, 1.7976931348623157e308, 2**40, 2**41, 60)]
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
    assert sorted(cfgs) == g["names"].tolist()
    for name, cfg in cfgs.items():
        line = canonical_config(cfg, 301 if name != "ls" else 69, 142)
        assert line == str(g[f"{name}__line"]), name
        buf = io.StringIO()
        write_csv(rows, buf, config_line=line)
        assert buf.getvalue() == str(g[f"{name}__csv"]), name
    buf = io.StringIO()
    write_csv(rows, buf)
    assert buf.getvalue() == str(g["noconfig__csv"])
    path = tmp_path / "rows.csv"
    path.write_text(str(g["c0__csv"]))
    line, back = read_csv(str(path))
    assert line == str(g["c0__line"])
    assert [(r.round, r.wall_seconds, r.grad_norm, r.f_value, r.bytes_up_cum, r.bytes_down_cum, r.ls_steps)
            for r in back] == [(r.round, r.wall_seconds, r.grad_norm, r.f_value, r.bytes_up_cum,
                                r.bytes_down_cum, r.ls_steps) for r in rows]
