"""Parity at the BASELINE stress shape c4 (d = 1024, n = 512, n_i = 2048,
dense Gaussian features, TopK k = 8192, lambda = 1e-4).

* P2 at shape: the oracle (f, gradient, packed Hessian) of a subset of c4's
  clients at x = 0 and at a random x, normwise 1e-10 per client.
* P5 at shape: one teacher-forced round of all 512 clients from a perturbed
  state; D, l_i and the index sets of sampled clients against the CPU
  oracle, the mean gradient of all 512 clients.
* P6: the first two c4 rounds (plus the final row) against the reference's
  own simulate (tests/golden/simulate_c4.npz, oracle/make_golden.py gen_c4).

The shards are regenerated here from their seed (numpy default_rng,
data.gaussian_shards): 8.6 GB of host memory for the whole set.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from oracle import fednl_oracle as O
from paper_2410_08760_b200 import data as D
from paper_2410_08760_b200 import simulate
from paper_2410_08760_b200.engine import FedNLEngine

pytestmark = pytest.mark.gpu

C4 = D.BASELINE_CONFIGS["c4"]


def normwise(got, want, scale=None):
    want = np.asarray(want)
    s = np.max(np.abs(want)) if scale is None else scale
    return float(np.max(np.abs(np.asarray(got) - want))) / max(s, 1e-300)


@pytest.fixture(scope="module")
def c4_shards():
    return D.baseline_shards("c4")


def test_oracle_at_c4_shape():
    """f, gradient and the packed Hessian of c4 clients (the first 6 of the
    c4 stream: same bytes as in the full set) at x = 0 and a random x."""
    shards = D.gaussian_shards(C4["d"], 6, C4["ni"], C4["lam"], seed=1)
    d = shards[0].dim
    cfg = D.baseline_run_config("c4", rounds=1)
    rng = np.random.default_rng(7)
    for x in (np.zeros(d), 0.05 * rng.standard_normal(d)):
        with FedNLEngine(cfg, d, len(shards), shards[0].n_samples) as eng:
            eng.upload([s.bmat for s in shards], [s.lam for s in shards])
            f, g, h = eng.oracle_eval(x)
        for c, s in enumerate(shards):
            ev = O.local_eval(s.bmat, s.lam, x)
            assert abs(f[c] - ev.f) <= 1e-12 * abs(ev.f), c
            assert normwise(g[c], ev.grad) <= 1e-10, c
            assert normwise(h[c], ev.hess) <= 1e-10, c


def test_teacher_forced_round_at_c4_shape(c4_shards):
    """One FedNL round of all 512 clients from a forced state (x random,
    client estimates lambda I plus a random sparse perturbation): the GPU's
    D_i, l_i and TopK index sets of sampled clients match the CPU oracle
    (D at 1e-10 of max |H_i|; index sets equal up to k-th-boundary ties), and
    the mean gradient of all 512 clients matches at 1e-10."""
    shards = c4_shards
    cfg = D.baseline_run_config("c4", rounds=1)
    d, n = shards[0].dim, len(shards)
    w = d * (d + 1) // 2
    k = cfg.compressor.k
    rng = np.random.default_rng(11)
    x = 0.03 * rng.standard_normal(d)
    diag = O.diag_positions(d)
    h_cli = np.zeros((n, w))
    h_cli[:, diag] = C4["lam"]
    for c in range(n):  # a sparse perturbation per client
        pos = rng.choice(w, 64, replace=False)
        h_cli[c, pos] += 1e-3 * rng.standard_normal(64)
    eng = FedNLEngine(cfg, d, n, shards[0].n_samples)
    eng.upload([s.bmat for s in shards], [s.lam for s in shards])
    eng.init_state()
    eng.set_x(x)
    eng.set_client_hest(h_cli)
    eng.run_rounds(1, first_round=0)
    _, cli_shift = eng.round_scalars()
    mg, _ = eng.round_grads()
    want_g = np.zeros(d)
    for c in range(n):
        m = shards[c].bmat.T @ x
        want_g += O.grad_from_sigmoid(shards[c].bmat, O.sigmoid(m), x, shards[c].lam)
    assert normwise(mg, want_g / n) <= 1e-10
    for c in (0, 1, 257, 511):
        ev = O.local_eval(shards[c].bmat, shards[c].lam, x)
        ref_d = ev.hess - h_cli[c]
        dv = eng.round_diff(c)
        assert np.max(np.abs(dv - ref_d)) <= 1e-10 * np.max(np.abs(ev.hess)), c
        assert abs(cli_shift[c] - O.frob(ref_d, d)) <= 1e-10 * O.frob(ref_d, d), c
        idx, val = eng.round_delta(c)
        ref_idx = O.compress_packed(ref_d, d, "topk", k, O.round_stream(cfg.run_seed, c, 0)).indices
        sym = np.setxor1d(idx, ref_idx)
        if sym.size:  # k-th-boundary ties only
            for dvv in (dv, ref_d):
                kth = np.sort(np.abs(dvv))[::-1][k - 1]
                assert np.all(np.abs(np.abs(dvv[sym]) - kth) <= 4 * np.spacing(kth)), c
        assert np.array_equal(val, dv[idx])
    eng.close()


def test_c4_rounds_match_reference(c4_shards):
    """Rows 0, 1 and the final row of a 2-round c4 run against the
    reference's simulate: grad_norm at 1e-10, f at 1e-12, byte counters
    exact."""
    from test_gpu_parity import _rows_close

    cfg = D.baseline_run_config("c4", rounds=2)
    rows = simulate(cfg, c4_shards)
    _rows_close(rows, golden("simulate_c4.npz"), ["c4_r2"])
