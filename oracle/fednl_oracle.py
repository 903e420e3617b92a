"""CPU oracle for the simulated FedNL round — TEST INFRASTRUCTURE, NOT PRODUCT.

This module restates, in numpy, the reference algorithm of
arxiv/paper_2410_08760 (`/root/reference/pkg/src/fednl`) for the one hot
path this repository accelerates: the simulated FedNL / FedNL-LS / FedNL-PP
round.  It exists only to CHECK the CUDA path:

* `tests/` compare the CUDA library against it on seeded inputs;
* `__graft_entry__.smoke()` checks one small round against it;
* `bench.py` times it as the CPU baseline (`cpu_baseline`, `--impl reference`).

Nothing under `paper_2410_08760_b200/` imports it; the product path has no CPU
fallback.

Pinning: `oracle/make_golden.py` runs the reference itself (imported from
/root/reference in the build container) and writes `tests/golden/*.npz`;
`tests/test_oracle_golden.py` checks this restatement against every one of
those vectors (SplitMix64 seed-0 stream, randrange / partial-shuffle draws,
compressor outputs on fixed inputs, oracle values, Cholesky solves, and whole
`simulate` trajectories incl. byte counters) — bit-for-bit where the reference
is deterministic on this host (OPENBLAS_NUM_THREADS=1).

State is kept in packed upper-triangle form (column-wise, t = j(j+1)/2 + i;
`linalg.py:54-58`); every floating-point expression that the reference
evaluates is evaluated here with the same numpy/BLAS call on the same layout
so the two agree bitwise on one host.
"""

from __future__ import annotations

import math
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

# --------------------------------------------------------------------------
# SplitMix64 (rng.py:26-136)

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15  # rng.py:26
MIX1 = 0xBF58476D1CE4E5B9  # rng.py:27
MIX2 = 0x94D049BB133111EB  # rng.py:28
TAG_SHUFFLE = 0x8000000000000001  # rng.py:32
TAG_SYNTH = 0x8000000000000002  # rng.py:33
TAG_MASTER = 0x8000000000000003  # rng.py:34

_U64 = np.uint64


def scramble(z: int) -> int:
    """SplitMix64 output function of a *state* value (rng.py:58-63 body)."""
    z = ((z ^ (z >> 30)) * MIX1) & MASK64
    z = ((z ^ (z >> 27)) * MIX2) & MASK64
    return z ^ (z >> 31)


def mix64(z: int) -> int:
    """rng.py:37-42: advance-by-golden then scramble."""
    return scramble((z + GOLDEN) & MASK64)


class SplitMix64:
    """Counter-based SplitMix64 stream (rng.py:45-118).

    Draw i (1-based) of a stream seeded with s is scramble(s + i*GOLDEN).
    """

    def __init__(self, seed: int):
        self.state = seed & MASK64
        self.seed0 = self.state

    def next_u64(self) -> int:  # rng.py:58-63
        self.state = (self.state + GOLDEN) & MASK64
        return scramble(self.state)

    def u64_block(self, n: int) -> np.ndarray:  # rng.py:65-76
        if n < 0:
            raise ValueError("negative draw count")
        ctr = _U64(self.state) + _U64(GOLDEN) * np.arange(1, n + 1, dtype=np.uint64)
        self.state = (self.state + n * GOLDEN) & MASK64
        z = (ctr ^ (ctr >> _U64(30))) * _U64(MIX1)
        z = (z ^ (z >> _U64(27))) * _U64(MIX2)
        return z ^ (z >> _U64(31))

    def next_f64(self) -> float:  # rng.py:78-80
        return (self.next_u64() >> 11) * 2.0**-53

    def f64_block(self, n: int) -> np.ndarray:  # rng.py:82-84
        return (self.u64_block(n) >> _U64(11)).astype(np.float64) * 2.0**-53

    def randrange(self, bound: int) -> int:  # rng.py:86-97
        if bound <= 0:
            raise ValueError("bound must be positive")
        reject_below = (1 << 64) % bound
        u = self.next_u64()
        while u < reject_below:
            u = self.next_u64()
        return u % bound

    def shuffle(self, arr) -> None:  # rng.py:99-104
        for i in range(len(arr) - 1, 0, -1):
            j = self.randrange(i + 1)
            arr[i], arr[j] = arr[j], arr[i]

    def partial_shuffle_prefix(self, n: int, k: int) -> np.ndarray:  # rng.py:106-118
        if not 0 <= k <= n:
            raise ValueError("need 0 <= k <= n")
        # sparse pool: only touched slots are materialised
        pool: dict[int, int] = {}
        out = np.empty(k, dtype=np.int64)
        for i in range(k):
            j = i + self.randrange(n - i)
            vi, vj = pool.get(i, i), pool.get(j, j)
            pool[i], pool[j] = vj, vi
            out[i] = vj
        return out


def round_seed(run_seed: int, cid: int, rnd: int) -> int:  # rng.py:121-127
    if not 0 <= cid < (1 << 32):
        raise ValueError("client_id out of u32 range")
    if not 0 <= rnd < (1 << 32):
        raise ValueError("round out of u32 range")
    return mix64(run_seed ^ ((cid << 32) | rnd))


def round_stream(run_seed: int, cid: int, rnd: int) -> SplitMix64:  # rng.py:130-131
    return SplitMix64(round_seed(run_seed, cid, rnd))


def named_stream(run_seed: int, tag: int) -> SplitMix64:  # rng.py:134-136
    return SplitMix64(mix64(run_seed ^ tag))


# --------------------------------------------------------------------------
# packed layout (linalg.py:49-106)


def packed_len(d: int) -> int:
    return d * (d + 1) // 2


_TRI: dict[int, tuple[np.ndarray, np.ndarray, np.ndarray]] = {}


def tri(d: int):
    """(rows, cols, weights) of the packed enumeration (linalg.py:73-88)."""
    got = _TRI.get(d)
    if got is None:
        cols = np.repeat(np.arange(d), np.arange(1, d + 1))
        rows = np.arange(packed_len(d)) - cols * (cols + 1) // 2
        got = (rows, cols, np.where(rows == cols, 1.0, 2.0))
        _TRI[d] = got
    return got


def to_dense(pk: np.ndarray, d: int) -> np.ndarray:
    """Symmetric F-order matrix from a packed vector (linalg.py:98-106)."""
    rows, cols, _ = tri(d)
    out = np.zeros((d, d), order="F")
    out[rows, cols] = pk
    out[cols, rows] = pk
    return out


def pack_upper(m: np.ndarray) -> np.ndarray:
    """Packed upper triangle, column-wise (linalg.py:91-95)."""
    rows, cols, _ = tri(m.shape[0])
    return np.ascontiguousarray(m[rows, cols])


def diag_positions(d: int) -> np.ndarray:
    j = np.arange(d)
    return j * (j + 1) // 2 + j


def frob(pk: np.ndarray, d: int) -> float:
    """Weighted Frobenius norm from the upper triangle (linalg.py:139-148)."""
    w = tri(d)[2]
    return math.sqrt(float(np.dot(w * pk, pk)))


# --------------------------------------------------------------------------
# logistic oracle (oracle.py:64-139)


def sigmoid(m: np.ndarray) -> np.ndarray:  # oracle.py:64-71
    out = np.empty_like(m)
    nonneg = m >= 0
    out[nonneg] = 1.0 / (1.0 + np.exp(-m[nonneg]))
    e = np.exp(m[~nonneg])
    out[~nonneg] = e / (1.0 + e)
    return out


def margins(bmat: np.ndarray, x: np.ndarray) -> np.ndarray:  # oracle.py:80
    out = np.zeros(bmat.shape[1])
    np.matmul(bmat.T, x, out=out)
    return out


def f_from_margins(m: np.ndarray, x: np.ndarray, lam: float) -> float:  # oracle.py:95-105
    loss = np.empty_like(m)
    nonneg = m >= 0
    loss[nonneg] = np.log1p(np.exp(-m[nonneg]))
    loss[~nonneg] = -m[~nonneg] + np.log1p(np.exp(m[~nonneg]))
    return float(np.sum(loss)) / len(m) + 0.5 * lam * float(np.dot(x, x))


def grad_from_sigmoid(bmat, sig, x, lam) -> np.ndarray:  # oracle.py:108-121
    g = np.zeros(bmat.shape[0])
    np.matmul(bmat, (sig - 1.0) / bmat.shape[1], out=g)
    g += lam * x
    return g


def hess_packed_from_sigmoid(bmat, sig, lam) -> np.ndarray:  # oracle.py:124-139
    d, ni = bmat.shape
    full = np.zeros((d, d), order="F")
    np.matmul(bmat * (sig * (1.0 - sig) / ni), bmat.T, out=full)
    rows, cols, _ = tri(d)
    pk = np.ascontiguousarray(full[rows, cols])
    pk[diag_positions(d)] += lam
    return pk


@dataclass
class LocalEval:
    """Everything the oracle yields at one point for one client."""

    f: float
    grad: np.ndarray
    hess: np.ndarray | None  # packed


def local_eval(bmat, lam, x, need_hess=True, need_f=True) -> LocalEval:
    m = margins(bmat, x)
    sig = sigmoid(m)
    return LocalEval(
        f=f_from_margins(m, x, lam) if need_f else float("nan"),
        grad=grad_from_sigmoid(bmat, sig, x, lam),
        hess=hess_packed_from_sigmoid(bmat, sig, lam) if need_hess else None,
    )


# --------------------------------------------------------------------------
# compressors (compressors.py:41-393, 465-482)

KINDS = ("identity", "topk", "toplek", "randk", "randseqk", "natural")
NEEDS_K = {"topk", "toplek", "randk", "randseqk"}


@dataclass
class Delta:
    """Compressed packed delta (compressors.py:101-120)."""

    kind: str
    d: int
    values: np.ndarray
    indices: np.ndarray | None  # uint32 ascending, None for dense kinds
    seed_tag: int | None = None

    @property
    def count(self) -> int:
        return len(self.values)


def _empty(kind: str, d: int) -> Delta:  # compressors.py:123-129
    return Delta(kind, d, np.zeros(0), np.zeros(0, dtype=np.uint32))


def check_k(kind: str, k: int | None, w: int) -> None:  # compressors.py:70-80
    if kind in NEEDS_K:
        if k is None:
            raise ValueError(f"compressor {kind} requires k")
        if not 1 <= k <= w:
            raise ValueError(f"k={k} out of range [1, {w}] for {kind}")


def desc_order(keys: np.ndarray) -> np.ndarray:
    """Descending by key, ties to the smaller position (compressors.py:139-141)."""
    return np.lexsort((np.arange(len(keys)), -keys))


def numpy_pairwise_sum(a: np.ndarray) -> float:
    """numpy's float64 add.reduce order (pairwise, 8-way unrolled leaves of
    <=128); what `np.sum(sorted_energies)` at compressors.py:189 evaluates.
    Used by tests to document the order the CUDA TopLEK kernel replicates."""
    n = len(a)
    if n < 8:
        acc = 0.0
        for v in a:
            acc += float(v)
        return acc
    if n <= 128:
        r = [float(v) for v in a[:8]]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] += float(a[i + j])
            i += 8
        acc = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            acc += float(a[i])
            i += 1
        return acc
    half = n // 2
    half -= half % 8
    return numpy_pairwise_sum(a[:half]) + numpy_pairwise_sum(a[half:])


def toplek_plan(sorted_energy: np.ndarray, k: int) -> tuple[int, int, float]:
    """Two-prefix mixing law (compressors.py:179-207)."""
    w = len(sorted_energy)
    total = float(np.sum(sorted_energy))
    if total <= 0.0:
        raise ValueError("toplek plan needs positive total energy")
    target = k / w
    shares = np.cumsum(sorted_energy) / total
    hi = int(np.searchsorted(shares, target))
    if hi >= k:
        return k, k, 1.0
    hi += 1
    lo = hi - 1
    s_lo = 0.0 if lo == 0 else float(shares[lo - 1])
    s_hi = float(shares[hi - 1])
    if s_hi <= s_lo or s_hi <= target:
        return hi, hi, 1.0
    p = (s_hi - target) / (s_hi - s_lo)
    return lo, hi, min(max(p, 0.0), 1.0)


def natural_round(vals: np.ndarray, prg: SplitMix64) -> np.ndarray:
    """Stochastic power-of-two rounding (compressors.py:289-336)."""
    tiny, huge = 2.0**-1022, 2.0**1023
    mag = np.abs(vals)
    low = np.zeros_like(mag)
    high = np.zeros_like(mag)
    p_up = np.zeros_like(mag)
    normal = (mag >= tiny) & (mag < huge)
    if np.any(normal):
        _, e = np.frexp(mag[normal])
        lo = np.ldexp(0.5, e)
        low[normal] = lo
        high[normal] = np.ldexp(1.0, e)
        p_up[normal] = (mag[normal] - lo) / lo
    sub = (mag > 0.0) & (mag < tiny)
    if np.any(sub):
        high[sub] = tiny
        p_up[sub] = mag[sub] / tiny
    big = mag >= huge
    if np.any(big):
        low[big] = huge
        high[big] = huge
    u = prg.f64_block(len(vals))
    out = np.where(u < p_up, high, low)
    return np.where(vals < 0.0, -out, out)


def compress_packed(
    pk: np.ndarray, d: int, kind: str, k: int | None, prg: SplitMix64,
    topk_weighted: bool = False,
) -> Delta:
    """Dispatch of compressors.py:350-370 on a packed difference."""
    w = packed_len(d)
    if w <= 0:
        raise ValueError("packed length must be positive")
    check_k(kind, k, w)
    if not np.all(np.isfinite(pk)):  # compressors.py:132-136
        raise ValueError("cannot compress a matrix with non-finite entries")
    if not np.any(pk != 0.0):
        return _empty(kind, d)
    weights = tri(d)[2]
    if kind == "identity":  # :154-160
        return Delta(kind, d, pk.copy(), None)
    if kind == "topk":  # :144-176
        key = weights * pk * pk if topk_weighted else np.abs(pk)
        idx = np.sort(desc_order(key)[:k])
        return Delta(kind, d, pk[idx].copy(), idx.astype(np.uint32))
    if kind == "toplek":  # :210-233
        energy = weights * pk * pk
        order = desc_order(energy)
        lo, hi, p_lo = toplek_plan(energy[order], k)
        t = lo if prg.next_f64() < p_lo else hi
        idx = np.sort(order[:t])
        return Delta(kind, d, pk[idx].copy(), idx.astype(np.uint32))
    if kind in ("randk", "randseqk"):  # :252-272
        seed = prg.seed0
        if kind == "randk":
            idx = np.sort(prg.partial_shuffle_prefix(w, k))
        else:
            start = prg.randrange(w)
            idx = np.sort((start + np.arange(k, dtype=np.int64)) % w)
        return Delta(kind, d, pk[idx] * (w / k), idx.astype(np.uint32), seed)
    if kind == "natural":  # :339-347
        return Delta(kind, d, natural_round(pk, prg), None)
    raise ValueError(f"unknown compressor kind {kind!r}")


def apply_packed(h: np.ndarray, delta: Delta, scale: float) -> None:
    """h += scale * delta on packed storage (compressors.py:373-393)."""
    if delta.count == 0:
        return
    if delta.indices is None:
        h += scale * delta.values
    else:
        h[delta.indices] += scale * delta.values


def wire_bytes(delta: Delta, reconstruct: bool) -> int:  # compressors.py:465-482
    if delta.count == 0:
        return 0
    w = packed_len(delta.d)
    if delta.kind == "identity":
        return 8 * w
    if delta.kind == "natural":
        return (12 * w + 7) // 8
    if delta.kind in ("randk", "randseqk") and reconstruct:
        return 8 + 8 * delta.count
    return 12 * delta.count


# --------------------------------------------------------------------------
# master linear algebra (linalg.py:151-186)


class NotPD(Exception):
    def __init__(self, j: int, v: float):
        self.pivot_index, self.pivot_value = j, v
        super().__init__(
            f"matrix is not positive definite: pivot {j} has value {v:.6g}"
        )


def cholesky_lower(a: np.ndarray) -> np.ndarray:
    """Column-by-column Cholesky reading the upper triangle (linalg.py:151-173)."""
    d = a.shape[0]
    low = np.zeros((d, d), order="F")
    for j in range(d):
        piv = a[j, j] - np.dot(low[j, :j], low[j, :j])
        if not piv > 0.0 or not math.isfinite(piv):
            raise NotPD(j, float(piv))
        root = math.sqrt(piv)
        low[j, j] = root
        if j + 1 < d:
            low[j + 1:, j] = (a[j, j + 1:] - low[j + 1:, :j] @ low[j, :j]) / root
    return low


def cholesky_solve(a: np.ndarray, b: np.ndarray) -> np.ndarray:  # linalg.py:176-186
    low = cholesky_lower(a)
    d = low.shape[0]
    y = np.zeros(d)
    for i in range(d):
        y[i] = (b[i] - np.dot(low[i, :i], y[:i])) / low[i, i]
    x = np.zeros(d)
    for i in range(d - 1, -1, -1):
        x[i] = (y[i] - np.dot(low[i + 1:, i], x[i + 1:])) / low[i, i]
    return x


def shifted_solve(h_pk: np.ndarray, d: int, shift: float, rhs: np.ndarray) -> np.ndarray:
    """Solve (H + shift I) p = rhs from packed H (algorithms.py:361-367, option b)."""
    sysm = to_dense(h_pk, d)
    sysm[np.arange(d), np.arange(d)] += shift
    return cholesky_solve(sysm, rhs)


class EigenNotConverged(Exception):  # linalg.py:36-37
    pass


def jacobi_eigh(a: np.ndarray, max_sweeps: int = 30, tol_factor: float = 1e-12):
    """Cyclic Jacobi (linalg.py:189-245): rotations (p, q), p < q in row
    order, theta / t / c / s as the reference, |a_pq| <= 1e-300 skipped, a_pq
    set to zero; stop when sqrt(2 sum_{i<j} a_ij^2) <= tol * ||A||_F."""
    d = a.shape[0]
    work = np.array(a, dtype=np.float64, order="F", copy=True)
    vecs = np.eye(d, order="F")
    iu = np.triu_indices(d)
    wts = np.where(iu[0] == iu[1], 1.0, 2.0)
    norm = math.sqrt(float(np.sum(wts * work[iu] ** 2)))
    thresh = tol_factor * norm
    if d == 1 or norm == 0.0:
        return np.diag(work).copy(), vecs
    iu1 = np.triu_indices(d, 1)

    def off() -> float:
        o = work[iu1]
        return math.sqrt(2.0 * float(np.dot(o, o)))

    for _ in range(max_sweeps):
        if off() <= thresh:
            return np.diag(work).copy(), vecs
        for p in range(d - 1):
            for q in range(p + 1, d):
                apq = work[p, q]
                if abs(apq) <= 1e-300:
                    continue
                theta = (work[q, q] - work[p, p]) / (2.0 * apq)
                t = math.copysign(1.0, theta) / (abs(theta) + math.sqrt(theta * theta + 1.0))
                c = 1.0 / math.sqrt(t * t + 1.0)
                s = t * c
                rp, rq = work[p, :].copy(), work[q, :].copy()
                work[p, :] = c * rp - s * rq
                work[q, :] = s * rp + c * rq
                cp, cq = work[:, p].copy(), work[:, q].copy()
                work[:, p] = c * cp - s * cq
                work[:, q] = s * cp + c * cq
                work[p, q] = work[q, p] = 0.0
                vp, vq = vecs[:, p].copy(), vecs[:, q].copy()
                vecs[:, p] = c * vp - s * vq
                vecs[:, q] = s * vp + c * vq
    if off() <= thresh:
        return np.diag(work).copy(), vecs
    raise EigenNotConverged(f"Jacobi did not converge in {max_sweeps} sweeps (dim {d})")


def eigen_clamp_min(a: np.ndarray, floor: float) -> np.ndarray:  # linalg.py:248-259
    vals, vecs = jacobi_eigh(a)
    out = np.asfortranarray((vecs * np.maximum(vals, floor)) @ vecs.T)
    iu = np.triu_indices(a.shape[0], 1)
    out[iu[1], iu[0]] = out[iu]
    return out


def newton_direction(h_pk: np.ndarray, d: int, shift: float, rhs: np.ndarray, option: str,
                     mu: float) -> np.ndarray:  # algorithms.py:361-367
    if option == "a":
        return cholesky_solve(eigen_clamp_min(to_dense(h_pk, d), mu), rhs)
    return shifted_solve(h_pk, d, shift, rhs)


# --------------------------------------------------------------------------
# configuration helpers (algorithms.py:60-139)


def default_alpha(kind: str, k: int | None, w: int) -> float:  # algorithms.py:122-135
    check_k(kind, k, w)
    if kind == "identity":
        return 1.0
    if kind in ("topk", "toplek"):
        return 1.0 - math.sqrt(1.0 - k / w)
    if kind in ("randk", "randseqk"):
        return 1.0 / ((w / k - 1.0) + 1.0)
    return 1.0 / (0.125 + 1.0)


@dataclass
class OracleConfig:
    """Plain mirror of RunConfig's trajectory-defining fields."""

    algorithm: str = "fednl"
    kind: str = "identity"
    k: int | None = None
    topk_weighted: bool = False
    rounds: int = 100
    alpha: float | None = None
    lam: float = 1e-3
    ls_c: float = 0.49
    ls_gamma: float = 0.5
    tau: int | None = None
    run_seed: int = 0
    hessian_init: str = "lambda-identity"
    reconstruct_indices: bool = True
    stop_grad_norm: float | None = None
    option: str = "b"
    mu: float | None = None

    @property
    def effective_mu(self) -> float:  # algorithms.py:107-109
        return self.lam if self.mu is None else self.mu

    @classmethod
    def from_run_config(cls, cfg) -> "OracleConfig":
        comp = cfg.compressor
        return cls(
            algorithm=cfg.algorithm, kind=comp.kind.value if hasattr(comp.kind, "value") else str(comp.kind),
            k=comp.k, topk_weighted=comp.topk_weighted, rounds=cfg.rounds,
            alpha=cfg.alpha, lam=cfg.lam, ls_c=cfg.ls_c, ls_gamma=cfg.ls_gamma,
            tau=cfg.tau, run_seed=cfg.run_seed, hessian_init=cfg.hessian_init,
            reconstruct_indices=cfg.reconstruct_indices,
            stop_grad_norm=cfg.stop_grad_norm, option=cfg.option, mu=cfg.mu,
        )


def update_bytes(cfg: OracleConfig, d: int, delta_bytes: int) -> int:  # transport.py:383-388
    if cfg.algorithm == "fednl-pp":
        return 8 + 8 * d + delta_bytes
    return 8 * d + 8 + (8 if cfg.algorithm == "fednl-ls" else 0) + delta_bytes


def init_bytes(cfg: OracleConfig, d: int) -> int:  # transport.py:391-396
    size = 0
    if cfg.algorithm == "fednl-pp":
        size += 8 + 8 * d
    if cfg.hessian_init == "exact":
        size += 8 * packed_len(d)
    return size


class LineSearchFailed(Exception):
    def __init__(self, rnd: int):
        self.round = rnd
        super().__init__(f"line search failed at round {rnd}")


class Diverged(Exception):
    def __init__(self, rnd: int):
        self.round = rnd
        super().__init__(f"non-finite iterate after round {rnd}; run diverged")


LS_MAX = 60  # algorithms.py:38


@dataclass
class Row:
    round: int
    wall_seconds: float
    grad_norm: float
    f_value: float
    bytes_up_cum: int
    bytes_down_cum: int
    ls_steps: int


# --------------------------------------------------------------------------
# the simulated run on packed state (runtime.py:136-276, algorithms.py:170-442)


class OracleRun:
    """All n clients plus the master, state kept packed.

    `workers` only parallelises the per-client work (numpy releases the GIL
    in BLAS/lexsort); every cross-client reduction is in ascending cid, so
    results do not depend on it (runtime.py:132-167).
    """

    def __init__(self, cfg: OracleConfig, bmats: list[np.ndarray], lam: float | None = None,
                 workers: int = 1):
        if not bmats:
            raise ValueError("need at least one shard")
        self.cfg = cfg
        self.bmats = bmats
        self.n = len(bmats)
        self.d = bmats[0].shape[0]
        if any(b.shape[0] != self.d for b in bmats):
            raise ValueError("all shards must share one dimension")
        # per-client lambda (ClientShard.lam, oracle.py:33-46): one value or one per shard
        lam = cfg.lam if lam is None else lam
        self.lams = [float(v) for v in lam] if np.ndim(lam) else [float(lam)] * self.n
        self.lam = self.lams[0]
        self.w = packed_len(self.d)
        check_k(cfg.kind, cfg.k, self.w)
        self.alpha = default_alpha(cfg.kind, cfg.k, self.w) if cfg.alpha is None else cfg.alpha
        self.workers = max(1, workers)
        self.pool = ThreadPoolExecutor(self.workers) if self.workers > 1 else None
        d, n, w = self.d, self.n, self.w
        self.x = np.zeros(d)
        self.h_cli = np.zeros((n, w))
        self.h_mas = np.zeros(w)
        self.shift = 0.0
        self.gvec = np.zeros(d)
        self.cli_shift = np.zeros(n)
        self.cli_gvec = np.zeros((n, d))
        self.master_prg = named_stream(cfg.run_seed, TAG_MASTER)
        self.round = 0
        self.up = 0
        self.down = 0

    def close(self):
        if self.pool is not None:
            self.pool.shutdown(wait=True)
            self.pool = None

    def _map(self, fn, cids):
        if self.pool is None or len(cids) <= 1:
            return {c: fn(c) for c in cids}
        chunks = [cids[i::self.workers] for i in range(self.workers) if cids[i::self.workers]]
        futs = [self.pool.submit(lambda ch=ch: [(c, fn(c)) for c in ch]) for ch in chunks]
        out = {}
        for f in futs:
            out.update(f.result())
        return out

    # ---- init (algorithms.py:195-223, 331-349; runtime.py:223-231)
    def init(self) -> None:
        cfg, d, n = self.cfg, self.d, self.n
        diag = diag_positions(d)
        pp = cfg.algorithm == "fednl-pp"
        need_hess = cfg.hessian_init == "exact" or pp
        evals = self._map(lambda c: local_eval(self.bmats[c], self.lams[c], self.x,
                                               need_hess=need_hess, need_f=False)
                          if need_hess else None, list(range(n)))
        for c in range(n):
            if cfg.hessian_init == "zero":
                self.h_cli[c] = 0.0
            elif cfg.hessian_init == "lambda-identity":
                self.h_cli[c] = 0.0
                self.h_cli[c, diag] += self.lams[c]
            else:
                self.h_cli[c] = evals[c].hess
            if pp:
                diff = self.h_cli[c] - evals[c].hess
                self.cli_shift[c] = frob(diff, d)
                hd = to_dense(self.h_cli[c], d)
                self.cli_gvec[c] = hd @ self.x + self.cli_shift[c] * self.x - evals[c].grad
        if cfg.hessian_init == "lambda-identity":
            self.h_mas[diag] += cfg.lam
        elif cfg.hessian_init == "exact":
            acc = np.zeros(self.w)
            for c in range(n):
                acc += self.h_cli[c]
            acc /= n
            self.h_mas = acc
        if pp:
            s = 0.0
            g = np.zeros(d)
            for c in range(n):
                s += self.cli_shift[c]
                g += self.cli_gvec[c]
            self.shift = s / n
            self.gvec = g / n
        if cfg.algorithm == "fednl-pp" or cfg.hessian_init == "exact":
            self.down += 8 * d * n
            self.up += n * init_bytes(cfg, d)

    # ---- one client's FedNL round (algorithms.py:225-238)
    def client_round(self, cid: int, rnd: int):
        ev = local_eval(self.bmats[cid], self.lams[cid], self.x, need_hess=True,
                        need_f=True)
        diff = ev.hess - self.h_cli[cid]
        shift = frob(diff, self.d)
        delta = compress_packed(diff, self.d, self.cfg.kind, self.cfg.k,
                                round_stream(self.cfg.run_seed, cid, rnd),
                                self.cfg.topk_weighted)
        apply_packed(self.h_cli[cid], delta, self.alpha)
        return ev.grad, shift, delta, ev.f

    def mean_f(self, x) -> float:  # runtime.py:189-194
        vals = self._map(lambda c: f_from_margins(margins(self.bmats[c], x), x, self.lams[c]),
                         list(range(self.n)))
        tot = 0.0
        for c in range(self.n):
            tot += vals[c]
        return tot / self.n

    def mean_grad(self, x) -> np.ndarray:  # runtime.py:196-201
        vals = self._map(lambda c: grad_from_sigmoid(self.bmats[c], sigmoid(margins(self.bmats[c], x)),
                                                      x, self.lams[c]), list(range(self.n)))
        acc = np.zeros(self.d)
        for c in range(self.n):
            acc += vals[c]
        return acc / self.n

    def fold(self, deltas: dict) -> None:  # algorithms.py:369-372
        scale = self.alpha / self.n
        for c in sorted(deltas):
            apply_packed(self.h_mas, deltas[c], scale)

    def fednl_round(self, rnd: int) -> Row:
        """One FedNL or FedNL-LS round (runtime.py:255-268, algorithms.py:378-420)."""
        cfg, d, n = self.cfg, self.d, self.n
        ls = cfg.algorithm == "fednl-ls"
        x_k = self.x
        self.down += 8 * d * n
        res = self._map(lambda c: self.client_round(c, rnd), list(range(n)))
        deltas = {c: res[c][2] for c in range(n)}
        for c in range(n):
            self.up += update_bytes(cfg, d, wire_bytes(deltas[c], cfg.reconstruct_indices))
        grad = np.zeros(d)
        shift = 0.0
        for c in range(n):
            grad += res[c][0]
            shift += res[c][1]
        grad = grad / n
        shift = shift / n
        steps = 0
        if ls:
            f_now = 0.0
            for c in range(n):
                f_now += res[c][3]
            f_now /= n
            p = newton_direction(self.h_mas, d, shift, grad, cfg.option, cfg.effective_mu)
            dec = float(np.dot(grad, p))
            best = np.inf
            x_new = None
            for s in range(LS_MAX + 1):
                step = cfg.ls_gamma ** s
                trial = self.x - step * p
                self.down += 8 * d * n
                self.up += 8 * n
                ft = self.mean_f(trial)
                if ft <= f_now - cfg.ls_c * step * dec:
                    steps, x_new = s, trial
                    break
                best = min(best, ft)
            if x_new is None:
                raise LineSearchFailed(self.round)
            self.fold(deltas)
            self.x = x_new
            f_value = f_now
        else:
            f_value = self.mean_f(x_k)
            p = newton_direction(self.h_mas, d, shift, grad, cfg.option, cfg.effective_mu)
            self.fold(deltas)
            self.x = self.x - p
        self.round += 1
        if not np.all(np.isfinite(self.x)):
            raise Diverged(self.round)
        return Row(rnd, 0.0, float(np.linalg.norm(grad)), f_value, self.up, self.down, steps)

    # ---- FedNL-PP (runtime.py:236-253, algorithms.py:240-264, 422-442)
    def pp_client(self, cid: int, x_new: np.ndarray, rnd: int):
        ev = local_eval(self.bmats[cid], self.lams[cid], x_new, need_hess=True, need_f=False)
        diff = ev.hess - self.h_cli[cid]
        delta = compress_packed(diff, self.d, self.cfg.kind, self.cfg.k,
                                round_stream(self.cfg.run_seed, cid, rnd),
                                self.cfg.topk_weighted)
        apply_packed(self.h_cli[cid], delta, self.alpha)
        s_new = frob(self.h_cli[cid] - ev.hess, self.d)
        g_new = to_dense(self.h_cli[cid], self.d) @ x_new + s_new * x_new - ev.grad
        out = (delta, s_new - self.cli_shift[cid], g_new - self.cli_gvec[cid])
        self.cli_shift[cid] = s_new
        self.cli_gvec[cid] = g_new
        return out

    def pp_round(self, rnd: int) -> tuple[Row, bool]:
        cfg, d, n = self.cfg, self.d, self.n
        gn = float(np.linalg.norm(self.mean_grad(self.x)))
        fv = self.mean_f(self.x)
        if cfg.stop_grad_norm is not None and gn <= cfg.stop_grad_norm:
            return Row(rnd, 0.0, gn, fv, self.up, self.down, 0), True
        chosen = sorted(int(c) for c in self.master_prg.partial_shuffle_prefix(n, cfg.tau))
        x_new = shifted_solve(self.h_mas, d, self.shift, self.gvec)
        self.x = x_new
        if not np.all(np.isfinite(self.x)):
            raise Diverged(self.round)
        self.down += 8 * d * len(chosen)
        res = self._map(lambda c: self.pp_client(c, x_new, rnd), chosen)
        for c in chosen:
            self.up += update_bytes(cfg, d, wire_bytes(res[c][0], cfg.reconstruct_indices))
        for c in chosen:
            self.gvec = self.gvec + res[c][2] / n
            self.shift += res[c][1] / n
        self.fold({c: res[c][0] for c in chosen})
        self.round += 1
        return Row(rnd, 0.0, gn, fv, self.up, self.down, 0), False

    def run(self) -> list[Row]:
        """The whole `simulate` loop (runtime.py:176-276)."""
        cfg = self.cfg
        t0 = time.perf_counter()
        rows: list[Row] = []
        self.init()
        stopped = False
        for rnd in range(cfg.rounds):
            if cfg.algorithm == "fednl-pp":
                row, stop = self.pp_round(rnd)
                row.wall_seconds = time.perf_counter() - t0
                rows.append(row)
                if stop:
                    stopped = True
                    break
                continue
            row = self.fednl_round(rnd)
            row.wall_seconds = time.perf_counter() - t0
            rows.append(row)
            if cfg.stop_grad_norm is not None and row.grad_norm <= cfg.stop_grad_norm:
                stopped = True
                break
        if not stopped:
            gn = float(np.linalg.norm(self.mean_grad(self.x)))
            rows.append(Row(cfg.rounds, time.perf_counter() - t0, gn, self.mean_f(self.x),
                            self.up, self.down, 0))
        return rows


def simulate(cfg: OracleConfig, bmats: list[np.ndarray], lam: float | None = None,
             workers: int = 1) -> list[Row]:
    run = OracleRun(cfg, bmats, lam, workers)
    try:
        return run.run()
    finally:
        run.close()
