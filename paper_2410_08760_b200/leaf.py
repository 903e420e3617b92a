"""Device-backed leaf operations with the reference's leaf signatures.

These are the parity entry points of SURVEY §8(b): each runs the same CUDA
kernels the round graph uses, on injected inputs, through the C ABI.

* `compress(m, spec, prg)`            compressors.py:350-370
* `compress_packed_batch(...)`        the same over many clients at once
* `oracle_eval(shards, x)`            oracle.py:95-139 for every client
* `cholesky_solve(a, b)`              linalg.py:176-186 (via the shifted solve)
* `prg_*`                             rng.py draws generated on the device
"""

from __future__ import annotations

import ctypes as C
from functools import lru_cache

import numpy as np

from . import _lib
from .config import CompressedDelta, CompressorKind, CompressorSpec, RunConfig, packed_length
from .engine import FedNLEngine
from .rng import Prg


def _dim_from_packed(w: int) -> int:
    d = int((np.sqrt(8 * w + 1) - 1) // 2)
    while d * (d + 1) // 2 < w:
        d += 1
    if d * (d + 1) // 2 != w:
        raise ValueError("packed length does not match any dimension")
    return d


# TopK kernel variant of the compress engines (_lib.TOPK_PATH_*): results are
# identical by construction; the parity tests pin each variant in turn
TOPK_PATH = _lib.TOPK_PATH_AUTO


@lru_cache(maxsize=32)
def _compress_engine(d: int, n: int, kind: CompressorKind, k: int | None, weighted: bool,
                     topk_path: int = 0) -> FedNLEngine:
    cfg = RunConfig(compressor=CompressorSpec(kind, k=k, topk_weighted=weighted), alpha=1.0)
    return FedNLEngine(cfg, d, n, 1, topk_path=topk_path)


def _upper_packed(m: np.ndarray) -> np.ndarray:
    d = m.shape[0]
    iu = np.triu_indices(d)
    # column-wise packed order: t = j(j+1)/2 + i
    order = np.lexsort((iu[0], iu[1]))
    return np.ascontiguousarray(m[iu[0][order], iu[1][order]])


def compress_packed_batch(packed: np.ndarray, d: int, spec: CompressorSpec, seeds) -> list[CompressedDelta]:
    """Compress n packed differences; seeds[c] seeds client c's fresh stream."""
    w = packed_length(d)
    spec.validate(w)
    P = np.ascontiguousarray(packed, dtype=np.float64).reshape(-1, w)
    n = P.shape[0]
    eng = _compress_engine(d, n, spec.kind, spec.k, bool(spec.topk_weighted), TOPK_PATH)
    sd = np.array([int(s) & ((1 << 64) - 1) for s in seeds], dtype=np.uint64)
    idx, val, cnt, drw = eng.compress(P, sd)
    out = []
    dense = spec.kind in (CompressorKind.IDENTITY, CompressorKind.NATURAL)
    rand = spec.kind in (CompressorKind.RANDK, CompressorKind.RANDSEQK)
    for c in range(n):
        k = int(cnt[c])
        if k == 0:
            out.append(CompressedDelta(spec.kind, d, np.zeros(0), np.zeros(0, dtype=np.uint32)))
        elif dense:
            out.append(CompressedDelta(spec.kind, d, val[c].copy(), None))
        else:
            out.append(CompressedDelta(spec.kind, d, val[c, :k].copy(), idx[c, :k].copy(),
                                       int(sd[c]) if rand else None))
        out[-1].draws = int(drw[c])
    return out


def compress(m: np.ndarray, spec: CompressorSpec, prg: Prg) -> CompressedDelta:
    """compressors.py:350-370 on the device; advances `prg` by the draws used."""
    m = np.asarray(m, dtype=np.float64)
    if m.ndim == 2:
        d = m.shape[0]
        packed = _upper_packed(m)
    else:
        d = _dim_from_packed(m.shape[0])
        packed = m
    delta = compress_packed_batch(packed[None, :], d, spec, [prg.seed0])[0]
    for _ in range(delta.draws):
        prg.next_u64()
    return delta


def oracle_eval(shards, x: np.ndarray, hessian: bool = True):
    """(f [n], grad [n, d], packed Hessians [n, w] | None) of every client at x."""
    d, n, ni = shards[0].dim, len(shards), max(s.n_samples for s in shards)
    cfg = RunConfig(lam=shards[0].lam)
    with FedNLEngine(cfg, d, n, ni) as eng:
        eng.upload([s.bmat for s in shards], [s.lam for s in shards])
        return eng.oracle_eval(x, hessian=hessian)


@lru_cache(maxsize=8)
def _solve_engine(d: int) -> FedNLEngine:
    return FedNLEngine(RunConfig(), d, 1, 1)


def shifted_solve(h_packed: np.ndarray, d: int, shift: float, rhs: np.ndarray) -> np.ndarray:
    return _solve_engine(d).shifted_solve(h_packed, shift, rhs)


def cholesky_solve(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Solve a x = b for SPD a, reading only its upper triangle (linalg.py:176)."""
    a = np.asarray(a, dtype=np.float64)
    return shifted_solve(_upper_packed(a), a.shape[0], 0.0, b)


def prg_u64(seed: int, count: int) -> np.ndarray:
    out = np.zeros(count, dtype=np.uint64)
    _lib.check(_lib.load().fb_prg_u64(seed & ((1 << 64) - 1), count, _lib.ptr(out, C.c_uint64)),
               None, "fb_prg_u64")
    return out


def prg_randrange(seed: int, bounds, reps: int) -> tuple[np.ndarray, np.ndarray]:
    b = np.array([int(x) for x in bounds], dtype=np.uint64)
    out = np.zeros((len(b), reps), dtype=np.uint64)
    nxt = np.zeros(len(b), dtype=np.uint64)
    _lib.check(_lib.load().fb_prg_randrange(seed & ((1 << 64) - 1), _lib.ptr(b, C.c_uint64), len(b), reps,
                                            _lib.ptr(out, C.c_uint64), _lib.ptr(nxt, C.c_uint64)),
               None, "fb_prg_randrange")
    return out, nxt


def prg_partial_shuffle(seed: int, n: int, k: int) -> np.ndarray:
    out = np.zeros(k, dtype=np.int64)
    _lib.check(_lib.load().fb_prg_partial_shuffle(seed & ((1 << 64) - 1), n, k, _lib.ptr(out, C.c_int64)),
               None, "fb_prg_partial_shuffle")
    return out


def round_seeds(run_seed: int, n: int, rnd: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    _lib.check(_lib.load().fb_round_seeds(run_seed & ((1 << 64) - 1), n, rnd, _lib.ptr(out, C.c_uint64)),
               None, "fb_round_seeds")
    return out


def _unpack_symmetric(pk: np.ndarray, d: int) -> np.ndarray:
    iu = np.triu_indices(d)
    order = np.lexsort((iu[0], iu[1]))
    out = np.zeros((d, d), order="F")
    out[iu[0][order], iu[1][order]] = pk
    out[iu[1][order], iu[0][order]] = pk
    return out


def jacobi_eigh(a: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """linalg.py:189-245 on the device (parallel-order Jacobi, same rotation,
    threshold 1e-12 ||A||_F and 30-sweep cap): (eigenvalues, eigenvectors as
    columns), unsorted; EigenConvergenceError when the sweeps run out."""
    a = np.asarray(a, dtype=np.float64)
    d = a.shape[0]
    if a.shape != (d, d):
        raise ValueError("matrix must be square")
    _, vals, vecs = _solve_engine(d).eigen_clamp(_upper_packed(a), -np.inf, vectors=True)
    return vals, vecs


def eigen_clamp_min(a: np.ndarray, floor: float) -> np.ndarray:
    """linalg.py:248-259 on the device: the symmetric matrix with every
    eigenvalue below `floor` lifted to it (upper triangle mirrored)."""
    a = np.asarray(a, dtype=np.float64)
    d = a.shape[0]
    out, _, _ = _solve_engine(d).eigen_clamp(_upper_packed(a), float(floor))
    return _unpack_symmetric(out, d)
