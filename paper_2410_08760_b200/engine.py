"""FedNLEngine — one device context holding a whole simulated FedNL run.

Owns the C-ABI context (include/fednl_b200.h): shards in HBM, every client's
packed Hessian estimate, the master state and the captured round graph.
`runtime.simulate` drives it; tests use its state taps for teacher forcing.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .config import (
    KIND_CODE,
    CompressorKind,
    DivergenceError,
    EigenConvergenceError,
    LineSearchError,
    NotPositiveDefiniteError,
    RunConfig,
    packed_length,
    resolve_alpha,
)


@dataclass
class RoundBatch:
    """Per-round outputs of `FedNLEngine.run_rounds`."""

    grad_norm: np.ndarray
    f_value: np.ndarray
    ls_steps: np.ndarray
    entry_counts: np.ndarray  # [rounds, n] (-1 = did not participate)
    wall_ms: np.ndarray
    done: int


def _fb_config(cfg: RunConfig, d: int, n: int, ni: int, topk_path: int = 0,
               b_store: int = 0) -> _lib.FbConfig:
    w = packed_length(d)
    cfg.compressor.validate(w)
    c = _lib.FbConfig()
    c.d, c.n_clients, c.n_samples = d, n, ni
    c.algorithm = _lib.ALG_CODE[cfg.algorithm]
    c.kind = KIND_CODE[cfg.compressor.kind]
    c.k = cfg.compressor.k or 0
    c.topk_weighted = int(bool(cfg.compressor.topk_weighted))
    c.tau = cfg.tau or 0
    c.hessian_init = _lib.INIT_CODE[cfg.hessian_init]
    c.option = 1 if cfg.option == "a" else 0  # FB_OPTION_A / FB_OPTION_B
    c.mu = float(cfg.effective_mu)
    c.alpha = float(resolve_alpha(cfg, w))
    c.lam = float(cfg.lam)
    c.ls_c = float(cfg.ls_c)
    c.ls_gamma = float(cfg.ls_gamma)
    c.run_seed = int(cfg.run_seed)
    for s in range(61):  # gamma ** s exactly as the host evaluates it (algorithms.py:305)
        c.ls_steps_table[s] = cfg.ls_gamma ** s
    c.topk_path = int(topk_path)
    c.b_store = int(b_store)
    return c


class FedNLEngine:
    """Device-resident FedNL run.  Not re-entrant; one host thread.

    `n_samples` is the largest shard's sample count (shards may be ragged);
    `lam` is every shard's lambda unless `upload` is given per-shard values
    (the master's lambda-identity init uses cfg.lam, algorithms.py:334-335);
    `topk_path` pins a TopK kernel variant (_lib.TOPK_PATH_*; results are
    identical, tests use it to cover both); `b_store` = _lib.BSTORE_F64 keeps
    the margins-type passes on the fp64 design matrices (no compact copy;
    results identical, tests compare both)."""

    def __init__(self, cfg: RunConfig, d: int, n_clients: int, n_samples: int, lam: float | None = None,
                 topk_path: int = 0, b_store: int = 0):
        self.lib = _lib.load()
        self.cfg = cfg
        self.d, self.n, self.ni = d, n_clients, n_samples
        self.w = packed_length(d)
        fc = _fb_config(cfg, d, n_clients, n_samples, topk_path, b_store)
        self.default_lam = float(cfg.lam if lam is None else lam)
        self.alpha = fc.alpha
        h = C.c_void_p()
        rc = self.lib.fb_create(C.byref(fc), C.byref(h))
        if rc != _lib.FB_OK:
            msg = _lib.last_error(None)
            if rc == _lib.FB_ERR_INVALID:
                raise ValueError(msg)
            raise RuntimeError(f"fb_create failed (code {rc}): {msg}")
        self.h = h
        self.round = 0

    # ---------------------------------------------------------------- basics
    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.fb_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, rc: int, what: str) -> None:
        if rc == _lib.FB_OK:
            return
        st = self.status()
        msg = _lib.last_error(self.h)
        if rc == _lib.FB_ERR_NOT_PD:
            raise NotPositiveDefiniteError(st.pivot_index, st.pivot_value)
        if rc == _lib.FB_ERR_NONFINITE:
            raise ValueError("cannot compress a matrix with non-finite entries")
        if rc == _lib.FB_ERR_DIVERGED:
            raise DivergenceError(st.round)
        if rc == _lib.FB_ERR_LINE_SEARCH:
            raise LineSearchError(st.round, st.f_start, st.f_best)
        if rc == _lib.FB_ERR_EIGEN:
            raise EigenConvergenceError(msg or "Jacobi did not converge")
        if rc == _lib.FB_ERR_INVALID:
            raise ValueError(msg or what)
        raise RuntimeError(f"{what} failed (code {rc}): {msg}")

    def status(self) -> _lib.FbStatus:
        st = _lib.FbStatus()
        self.lib.fb_get_status(self.h, C.byref(st))
        return st

    # ------------------------------------------------------------------ data
    def set_shard(self, world: int, rank: int, nccl_id: bytes) -> None:
        """Own clients [rank*ceil(n/world), ...) and exchange with the other
        ranks over NCCL each round (before `upload`; FedNL only)."""
        if len(nccl_id) != 128:
            raise ValueError("nccl_id must be the 128-byte ncclUniqueId")
        buf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        self._check(self.lib.fb_set_shard(self.h, int(world), int(rank), buf), "fb_set_shard")
        self.world, self.rank = int(world), int(rank)

    def upload(self, bmats: list[np.ndarray], lams=None) -> None:
        """Shards (d x n_c each, n_c <= n_samples) and optionally their own
        lambdas (ClientShard.lam, oracle.py:33-46); another rank's shard may
        be None under sharding."""
        if len(bmats) != self.n:
            raise ValueError(f"expected {self.n} shards, got {len(bmats)}")
        keep = []
        ptrs = (C.POINTER(C.c_double) * self.n)()
        nis = np.full(self.n, self.ni, dtype=np.int32)
        lam = np.full(self.n, self.default_lam) if lams is None else np.asarray(lams, dtype=np.float64)
        if lam.shape != (self.n,):
            raise ValueError(f"expected {self.n} lambdas")
        lo, hi = shard_range(self.n, getattr(self, "world", 1), getattr(self, "rank", 0))
        for c, b in enumerate(bmats):
            if b is None and not lo <= c < hi:  # another rank's client (sharded)
                ptrs[c] = None
                continue
            if b.ndim != 2 or b.shape[0] != self.d or not 1 <= b.shape[1] <= self.ni:
                raise ValueError(f"shard {c} has shape {b.shape}, expected ({self.d}, 1..{self.ni})")
            a = np.asfortranarray(b, dtype=np.float64)
            keep.append(a)
            nis[c] = b.shape[1]
            ptrs[c] = a.ctypes.data_as(C.POINTER(C.c_double))
        self._check(self.lib.fb_upload_shards_ex(self.h, ptrs, _lib.ptr(nis, C.c_int32), _lib.ptr(lam)),
                    "fb_upload_shards_ex")

    def init_state(self, x0: np.ndarray | None = None) -> None:
        x = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
        self._check(self.lib.fb_init_state(self.h, _lib.ptr(x)), "fb_init_state")
        self.round = 0

    # ------------------------------------------------------------------- run
    def run_rounds(self, count: int, stop_grad_norm: float | None = None,
                   timed: bool = False, first_round: int | None = None) -> RoundBatch:
        r0 = self.round if first_round is None else first_round
        g = np.zeros(count)
        f = np.zeros(count)
        ls = np.zeros(count, dtype=np.int32)
        cnt = np.zeros((count, self.n), dtype=np.int32)
        wall = np.zeros(count)
        done = C.c_int32(0)
        rc = self.lib.fb_run_rounds(
            self.h, r0, count, -1.0 if stop_grad_norm is None else float(stop_grad_norm),
            int(timed), _lib.ptr(g), _lib.ptr(f), _lib.ptr(ls, C.c_int32),
            _lib.ptr(cnt, C.c_int32), _lib.ptr(wall), C.byref(done))
        self.round = r0 + done.value
        self._check(rc, "fb_run_rounds")
        k = done.value
        return RoundBatch(g[:k], f[:k], ls[:k], cnt[:k], wall[:k], k)

    def final_eval(self) -> tuple[float, float]:
        g, f = C.c_double(), C.c_double()
        self._check(self.lib.fb_final_eval(self.h, C.byref(g), C.byref(f)), "fb_final_eval")
        return g.value, f.value

    def profile(self) -> dict:
        p = _lib.FbProfile()
        self._check(self.lib.fb_get_profile(self.h, C.byref(p)), "fb_get_profile")
        return {k: getattr(p, k) for k, _ in p._fields_}

    # ------------------------------------------------------------ state taps
    def get_x(self) -> np.ndarray:
        x = np.zeros(self.d)
        self._check(self.lib.fb_get_x(self.h, _lib.ptr(x)), "fb_get_x")
        return x

    def set_x(self, x: np.ndarray) -> None:
        a = np.ascontiguousarray(x, dtype=np.float64)
        self._check(self.lib.fb_set_x(self.h, _lib.ptr(a)), "fb_set_x")

    def get_client_hest(self, c0: int = 0, c1: int | None = None) -> np.ndarray:
        c1 = self.n if c1 is None else c1
        out = np.zeros((c1 - c0, self.w))
        self._check(self.lib.fb_get_client_hest(self.h, c0, c1, _lib.ptr(out)), "fb_get_client_hest")
        return out

    def set_client_hest(self, values: np.ndarray, c0: int = 0) -> None:
        a = np.ascontiguousarray(values, dtype=np.float64).reshape(-1, self.w)
        self._check(self.lib.fb_set_client_hest(self.h, c0, c0 + a.shape[0], _lib.ptr(a)),
                    "fb_set_client_hest")

    def get_master_hest(self) -> np.ndarray:
        out = np.zeros(self.w)
        self._check(self.lib.fb_get_master_hest(self.h, _lib.ptr(out)), "fb_get_master_hest")
        return out

    def set_master_hest(self, values: np.ndarray) -> None:
        a = np.ascontiguousarray(values, dtype=np.float64)
        self._check(self.lib.fb_set_master_hest(self.h, _lib.ptr(a)), "fb_set_master_hest")

    def get_pp_state(self):
        shift = np.zeros(1)
        gvec = np.zeros(self.d)
        cs = np.zeros(self.n)
        cg = np.zeros((self.n, self.d))
        self._check(self.lib.fb_get_pp_state(self.h, _lib.ptr(shift), _lib.ptr(gvec), _lib.ptr(cs),
                                             _lib.ptr(cg)), "fb_get_pp_state")
        return float(shift[0]), gvec, cs, cg

    def round_diff(self, cid: int) -> np.ndarray:
        out = np.zeros(self.w)
        self._check(self.lib.fb_get_round_diff(self.h, cid, _lib.ptr(out)), "fb_get_round_diff")
        return out

    def round_delta(self, cid: int) -> tuple[np.ndarray | None, np.ndarray]:
        idx = np.zeros(self.w, dtype=np.uint32)
        val = np.zeros(self.w)
        cnt = C.c_int32()
        self._check(self.lib.fb_get_round_delta(self.h, cid, _lib.ptr(idx, C.c_uint32), _lib.ptr(val),
                                                C.byref(cnt)), "fb_get_round_delta")
        k = cnt.value
        kind = self.cfg.compressor.kind
        if kind in (CompressorKind.IDENTITY, CompressorKind.NATURAL):
            return None, val if k else np.zeros(0)
        return idx[:k].copy(), val[:k].copy()

    def round_scalars(self) -> tuple[dict, np.ndarray]:
        out = np.zeros(5)
        cs = np.zeros(self.n)
        self._check(self.lib.fb_get_round_scalars(self.h, _lib.ptr(out), _lib.ptr(cs)), "fb_get_round_scalars")
        keys = ("grad_norm", "f_mean", "shift_mean", "decrement", "xx")
        return dict(zip(keys, out.tolist())), cs

    def round_grads(self) -> tuple[np.ndarray, np.ndarray]:
        mg = np.zeros(self.d)
        cg = np.zeros((self.n, self.d))
        self._check(self.lib.fb_get_round_grads(self.h, _lib.ptr(mg), _lib.ptr(cg)), "fb_get_round_grads")
        return mg, cg

    # ------------------------------------------------------------- leaf ops
    def compress(self, diffs: np.ndarray, seeds: np.ndarray):
        """Compress n packed differences with per-client fresh streams."""
        D = np.ascontiguousarray(diffs, dtype=np.float64).reshape(self.n, self.w)
        sd = np.ascontiguousarray(seeds, dtype=np.uint64)
        idx = np.zeros((self.n, self.w), dtype=np.uint32)
        val = np.zeros((self.n, self.w))
        cnt = np.zeros(self.n, dtype=np.int32)
        drw = np.zeros(self.n, dtype=np.int32)
        rc = self.lib.fb_compress(self.h, _lib.ptr(D), _lib.ptr(sd, C.c_uint64), _lib.ptr(idx, C.c_uint32),
                                  _lib.ptr(val), _lib.ptr(cnt, C.c_int32), _lib.ptr(drw, C.c_int32))
        if rc == _lib.FB_ERR_NONFINITE:
            raise ValueError("cannot compress a matrix with non-finite entries")
        self._check(rc, "fb_compress")
        return idx, val, cnt, drw

    def oracle_eval(self, x: np.ndarray, hessian: bool = True):
        xa = np.ascontiguousarray(x, dtype=np.float64)
        f = np.zeros(self.n)
        g = np.zeros((self.n, self.d))
        h = np.zeros((self.n, self.w)) if hessian else None
        self._check(self.lib.fb_oracle_eval(self.h, _lib.ptr(xa), _lib.ptr(f), _lib.ptr(g), _lib.ptr(h)),
                    "fb_oracle_eval")
        return f, g, h

    def eigen_clamp(self, a_packed: np.ndarray, floor: float, vectors: bool = False):
        """eigen_clamp_min (linalg.py:248-259) of a packed symmetric matrix:
        (clamped packed, eigenvalues, eigenvectors as columns | None)."""
        ap = np.ascontiguousarray(a_packed, dtype=np.float64).reshape(self.w)
        out = np.zeros(self.w)
        vals = np.zeros(self.d)
        vt = np.zeros((self.d, self.d)) if vectors else None
        self._check(self.lib.fb_eigen_clamp(self.h, _lib.ptr(ap), float(floor), _lib.ptr(out),
                                            _lib.ptr(vals), _lib.ptr(vt) if vectors else None),
                    "fb_eigen_clamp")
        return out, vals, (vt.T.copy() if vectors else None)

    def shifted_solve(self, h_packed: np.ndarray, shift: float, rhs: np.ndarray) -> np.ndarray:
        hp = np.ascontiguousarray(h_packed, dtype=np.float64)
        b = np.ascontiguousarray(rhs, dtype=np.float64)
        z = np.zeros(self.d)
        self._check(self.lib.fb_shifted_solve(self.h, _lib.ptr(hp), float(shift), _lib.ptr(b), _lib.ptr(z)),
                    "fb_shifted_solve")
        return z


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (rank 0 makes it; broadcast it to the other ranks)."""
    lib = _lib.load()
    buf = (C.c_uint8 * 128)()
    _lib.check(lib.fb_nccl_unique_id(buf), None, "fb_nccl_unique_id")
    return bytes(buf)


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Clients [lo, hi) owned by `rank` (fb_set_shard's partition)."""
    npr = (n + world - 1) // world
    lo = min(n, rank * npr)
    return lo, min(n, lo + npr)


def fp64_peak() -> tuple[float, float]:
    """(DMMA TFLOP/s, DFMA TFLOP/s) measured on the current device."""
    lib = _lib.load()
    a, b = C.c_double(), C.c_double()
    _lib.check(lib.fb_fp64_peak(C.byref(a), C.byref(b)), None, "fb_fp64_peak")
    return a.value, b.value
