"""Client shards and synthetic input builders (host side, one-time, untimed).

`ClientShard` mirrors reference oracle.py:33-46: a d x n_i column-major
design matrix whose column j is label_j * (features_j, 1) — intercept last,
label absorbed.  The builders follow the reference's sharding conventions
(data.py:160-213: TAG_SHUFFLE Fisher-Yates over rows, equal shards of
floor(m/n) rows, remainder dropped) so both implementations receive the same
bytes.  The BASELINE generators are the SURVEY §8(d) stand-ins for the
W8A / A9A / Phishing shapes (those datasets are not available here).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .rng import TAG_SHUFFLE, TAG_SYNTH, Prg, derive_stream


@dataclass
class ClientShard:
    """One client's slice of the dataset, labels absorbed into columns."""

    bmat: np.ndarray  # d x n_i, column-major
    lam: float

    @property
    def dim(self) -> int:
        return self.bmat.shape[0]

    @property
    def n_samples(self) -> int:
        return self.bmat.shape[1]


def shard_permutation(m: int, n_clients: int, run_seed: int) -> tuple[np.ndarray, int]:
    """Row permutation + rows per client (data.py:160-172)."""
    per_client = m // n_clients
    if per_client < 1:
        raise ValueError(f"{m} samples cannot feed {n_clients} clients")
    perm = np.arange(m, dtype=np.int64)
    derive_stream(run_seed, TAG_SHUFFLE).shuffle(perm)
    return perm, per_client


def shards_from_dense(feats: np.ndarray, labels: np.ndarray, n_clients: int,
                      run_seed: int, lam: float, shuffle: bool = True) -> list[ClientShard]:
    """Dense (m, nf) features + {-1,+1} labels -> absorbed F-order shards.

    Equivalent to reference augment_and_shard (data.py:186-213) for a dataset
    whose sparse rows hold exactly the nonzeros of `feats`.
    """
    m, nf = feats.shape
    seen = set(np.unique(labels).tolist())
    if not seen <= {-1.0, 1.0}:
        raise ValueError(f"labels must be normalized to -1/+1, got {sorted(seen)}")
    if shuffle:
        perm, per = shard_permutation(m, n_clients, run_seed)
    else:
        per = m // n_clients
        perm = np.arange(m, dtype=np.int64)
    out = []
    for cid in range(n_clients):
        rows = perm[cid * per:(cid + 1) * per]
        b = np.empty((nf + 1, per), order="F")
        b[:nf, :] = feats[rows].T
        b[nf, :] = 1.0
        b *= labels[rows]
        out.append(ClientShard(bmat=b, lam=lam))
    return out


def generate_synthetic(num_features: int, m: int, seed: int,
                       margin_scale: float = 1.0) -> tuple[np.ndarray, np.ndarray]:
    """Dense uniform(-1,1) features with planted labels (data.py:257-277).

    Returns (features (m, nf), labels in {-1,+1}).
    """
    if num_features < 1 or m < 1:
        raise ValueError("need at least one feature and one sample")
    prg = derive_stream(seed, TAG_SYNTH)
    x_true = 2.0 * prg.f64_block(num_features) - 1.0
    feats = 2.0 * prg.f64_block(m * num_features).reshape(m, num_features) - 1.0
    noise = 2.0 * prg.f64_block(m) - 1.0
    score = margin_scale * (feats @ x_true) + noise
    return feats, np.where(score >= 0.0, 1.0, -1.0)


def make_shards(num_features: int, m: int, n: int, seed: int, lam: float = 1e-3):
    """The reference tests' fixture builder (test_runtime.py:34-37)."""
    feats, labels = generate_synthetic(num_features, m, seed)
    return shards_from_dense(feats, labels, n, run_seed=seed, lam=lam)


# ---------------------------------------------------------------- BASELINE


BASELINE_CONFIGS = {
    # shapes of the paper's W8A / A9A / Phishing runs
    "c0": dict(d=301, n=142, ni=350, gen="binary", density=0.04, p_pos=0.3, lam=1e-3,
               algorithm="fednl", kind="topk", k=2408, alpha=1.0, rounds=100),
    "c1": dict(d=124, n=80, ni=407, gen="binary", density=0.11, p_pos=0.24, lam=1e-3,
               algorithm="fednl", kind="randseqk", k=992, alpha=None, rounds=200),
    "c2": dict(d=69, n=100, ni=110, gen="binary", density=0.44, p_pos=0.5, lam=1e-3,
               algorithm="fednl-ls", kind="toplek", k=69, alpha=None, rounds=200),
    "c3": dict(d=301, n=142, ni=350, gen="binary", density=0.04, p_pos=0.3, lam=1e-3,
               algorithm="fednl-pp", kind="randk", k=301, alpha=None, rounds=500, tau=12),
    "c4": dict(d=1024, n=512, ni=2048, gen="gaussian", lam=1e-4,
               algorithm="fednl", kind="topk", k=8192, alpha=None, rounds=50),
}


def binary_shards(d: int, n: int, ni: int, density: float, p_pos: float, lam: float,
                  seed: int = 1) -> list[ClientShard]:
    """Sparse-binary stand-in: Prg(seed) features then labels."""
    m = n * ni
    prg = Prg(seed)
    feats = (prg.f64_block(m * (d - 1)).reshape(m, d - 1) < density).astype(np.float64)
    labels = np.where(prg.f64_block(m) < p_pos, 1.0, -1.0)
    return shards_from_dense(feats, labels, n, run_seed=seed, lam=lam)


def gaussian_shards(d: int, n: int, ni: int, lam: float, seed: int = 1) -> list[ClientShard]:
    """Dense Gaussian stress input (c4): y = sign(w*.a + eps), eps ~ N(0, 0.1 var)."""
    g = np.random.default_rng(seed)
    m = n * ni
    wstar = g.standard_normal(d - 1) / np.sqrt(d)
    out = []
    for cid in range(n):
        a = g.standard_normal((d - 1, ni))
        y = np.sign(wstar @ a + g.normal(0.0, np.sqrt(0.1), ni))
        y[y == 0] = 1.0
        b = np.empty((d, ni), order="F")
        b[:d - 1] = a
        b[d - 1] = 1.0
        b *= y
        out.append(ClientShard(bmat=b, lam=lam))
    del m
    return out


def baseline_shards(name: str, seed: int = 1) -> list[ClientShard]:
    c = BASELINE_CONFIGS[name]
    if c["gen"] == "binary":
        return binary_shards(c["d"], c["n"], c["ni"], c["density"], c["p_pos"], c["lam"], seed)
    return gaussian_shards(c["d"], c["n"], c["ni"], c["lam"], seed)


def baseline_run_config(name: str, rounds: int | None = None, run_seed: int = 1):
    from .config import CompressorKind, CompressorSpec, RunConfig

    c = BASELINE_CONFIGS[name]
    return RunConfig(
        algorithm=c["algorithm"],
        compressor=CompressorSpec(CompressorKind(c["kind"]), k=c["k"]),
        rounds=c["rounds"] if rounds is None else rounds,
        alpha=c["alpha"],
        lam=c["lam"],
        tau=c.get("tau"),
        run_seed=run_seed,
    )


# the reference's data-module names for real datasets (data.py:31-254)
from .ingest import (  # noqa: E402
    ParseError,
    RawDataset,
    augment_and_shard,
    load_client_shard,
    load_libsvm,
    normalize_labels,
    parse_libsvm,
    split_rows,
    write_libsvm,
)
