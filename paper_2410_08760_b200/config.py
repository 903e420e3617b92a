"""Run configuration and message types — the reference's public vocabulary.

Field names, defaults, validation messages and the resolved step size mirror
reference algorithms.py:35-167 and compressors.py:41-120 so that a caller of
`fednl.simulate(cfg, shards)` can switch imports and keep its code.
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field

import numpy as np

ALGORITHMS = ("fednl", "fednl-ls", "fednl-pp")  # algorithms.py:35
OPTIONS = ("a", "b")  # algorithms.py:36
HESSIAN_INITS = ("lambda-identity", "zero", "exact")  # algorithms.py:37
LS_MAX_BACKTRACKS = 60  # algorithms.py:38


class CompressorKind(str, enum.Enum):
    """compressors.py:41-47."""

    IDENTITY = "identity"
    TOPK = "topk"
    TOPLEK = "toplek"
    RANDK = "randk"
    RANDSEQK = "randseqk"
    NATURAL = "natural"


# device enum values (include/fednl_b200.h: FB_KIND_*)
KIND_CODE = {
    CompressorKind.IDENTITY: 0,
    CompressorKind.TOPK: 1,
    CompressorKind.TOPLEK: 2,
    CompressorKind.RANDK: 3,
    CompressorKind.RANDSEQK: 4,
    CompressorKind.NATURAL: 5,
}

_NEEDS_K = {CompressorKind.TOPK, CompressorKind.TOPLEK, CompressorKind.RANDK,
            CompressorKind.RANDSEQK}
_RAND = {CompressorKind.RANDK, CompressorKind.RANDSEQK}


@dataclass(frozen=True)
class CompressorSpec:
    """A compressor kind plus its budget k (compressors.py:59-98)."""

    kind: CompressorKind
    k: int | None = None
    topk_weighted: bool = False

    def validate(self, w: int) -> None:
        if self.kind in _NEEDS_K:
            if self.k is None:
                raise ValueError(f"compressor {self.kind.value} requires k")
            if not 1 <= self.k <= w:
                raise ValueError(f"k={self.k} out of range [1, {w}] for {self.kind.value}")
        if w <= 0:
            raise ValueError("packed length must be positive")

    def delta_fraction(self, w: int) -> float:
        if self.kind is CompressorKind.IDENTITY:
            return 1.0
        if self.kind in (CompressorKind.TOPK, CompressorKind.TOPLEK):
            return self.k / w
        raise ValueError(f"{self.kind.value} is not a contractive compressor")

    def omega(self, w: int) -> float:
        if self.kind is CompressorKind.IDENTITY:
            return 0.0
        if self.kind in _RAND:
            return w / self.k - 1.0
        if self.kind is CompressorKind.NATURAL:
            return 0.125
        raise ValueError(f"{self.kind.value} is not an unbiased compressor")


@dataclass
class CompressedDelta:
    """Packed compressed update (compressors.py:101-120)."""

    kind: CompressorKind
    d: int
    values: np.ndarray
    indices: np.ndarray | None = None
    seed_tag: int | None = None

    @property
    def entry_count(self) -> int:
        return len(self.values)


class LineSearchError(Exception):
    """Backtracking exhausted its cap (algorithms.py:41-49)."""

    def __init__(self, rnd: int, f_start: float, f_best: float):
        self.round = rnd
        super().__init__(
            f"line search failed at round {rnd}: started at f={f_start:.17g}, "
            f"best trial f={f_best:.17g} after {LS_MAX_BACKTRACKS} backtracks"
        )


class DivergenceError(Exception):
    """Non-finite iterate (algorithms.py:52-57)."""

    def __init__(self, rnd: int):
        self.round = rnd
        super().__init__(f"non-finite iterate after round {rnd}; run diverged")


class EigenConvergenceError(Exception):
    """Jacobi sweeps exhausted before the off-diagonal mass vanished (linalg.py:36-37)."""


class NotPositiveDefiniteError(Exception):
    """First Cholesky pivot that is <= 0 or not finite (linalg.py:24-33)."""

    def __init__(self, pivot_index: int, pivot_value: float):
        self.pivot_index = pivot_index
        self.pivot_value = pivot_value
        super().__init__(
            f"matrix is not positive definite: pivot {pivot_index} "
            f"has value {pivot_value:.6g}"
        )


@dataclass
class RunConfig:
    """Everything that determines a run's trajectory (algorithms.py:60-120)."""

    algorithm: str = "fednl"
    option: str = "b"
    compressor: CompressorSpec = field(
        default_factory=lambda: CompressorSpec(CompressorKind.IDENTITY)
    )
    rounds: int = 100
    alpha: float | None = None
    lam: float = 1e-3
    mu: float | None = None
    ls_c: float = 0.49
    ls_gamma: float = 0.5
    tau: int | None = None
    run_seed: int = 0
    hessian_init: str = "lambda-identity"
    reconstruct_indices: bool = True
    stop_grad_norm: float | None = None
    timeout_s: float = 30.0

    def validate(self, n_clients: int | None = None) -> None:
        if self.algorithm not in ALGORITHMS:
            raise ValueError(f"unknown algorithm {self.algorithm!r}")
        if self.option not in OPTIONS:
            raise ValueError(f"unknown option {self.option!r}")
        if self.hessian_init not in HESSIAN_INITS:
            raise ValueError(f"unknown hessian init {self.hessian_init!r}")
        if self.rounds < 0:
            raise ValueError("rounds must be >= 0")
        if self.lam < 0:
            raise ValueError("lambda must be >= 0")
        if not 0.0 < self.ls_c < 1.0:
            raise ValueError("line search c must be in (0, 1)")
        if not 0.0 < self.ls_gamma < 1.0:
            raise ValueError("line search gamma must be in (0, 1)")
        if self.algorithm == "fednl-pp":
            if self.tau is None:
                raise ValueError("fednl-pp requires tau")
            if n_clients is not None and not 1 <= self.tau <= n_clients:
                raise ValueError(f"tau={self.tau} out of range [1, {n_clients}]")
        if not 0 <= self.run_seed < (1 << 64):
            raise ValueError("seed must fit in 64 bits")

    @property
    def effective_mu(self) -> float:
        return self.lam if self.mu is None else self.mu

    @property
    def is_ls(self) -> bool:
        return self.algorithm == "fednl-ls"

    @property
    def is_pp(self) -> bool:
        return self.algorithm == "fednl-pp"

    def needs_init_exchange(self, n_clients: int) -> bool:
        return self.is_pp or self.hessian_init == "exact"


def default_alpha(spec: CompressorSpec, w: int) -> float:
    """Fold step size when `RunConfig.alpha` is None (algorithms.py:122-135)."""
    spec.validate(w)
    if spec.kind is CompressorKind.IDENTITY:
        return 1.0
    if spec.kind in (CompressorKind.TOPK, CompressorKind.TOPLEK):
        return 1.0 - math.sqrt(1.0 - spec.delta_fraction(w))
    return 1.0 / (spec.omega(w) + 1.0)


def resolve_alpha(cfg: RunConfig, w: int) -> float:
    return default_alpha(cfg.compressor, w) if cfg.alpha is None else cfg.alpha


@dataclass
class StepInfo:
    """What the master learned in one round (algorithms.py:275-281)."""

    grad_norm: float
    f_value: float | None = None
    ls_steps: int = 0


def packed_length(d: int) -> int:
    return d * (d + 1) // 2


def wire_size_bytes(kind: CompressorKind, d: int, count: int, reconstruct: bool) -> int:
    """Payload bytes of a delta block with `count` entries (compressors.py:465-482)."""
    if count == 0:
        return 0
    w = packed_length(d)
    if kind is CompressorKind.IDENTITY:
        return 8 * w
    if kind is CompressorKind.NATURAL:
        return (12 * w + 7) // 8
    if kind in _RAND and reconstruct:
        return 8 + 8 * count
    return 12 * count


def update_payload_size(cfg: RunConfig, d: int, delta_bytes: int) -> int:
    """CLIENT_UPDATE payload bytes (transport.py:383-388)."""
    if cfg.is_pp:
        return 8 + 8 * d + delta_bytes
    return 8 * d + 8 + (8 if cfg.is_ls else 0) + delta_bytes


def init_response_size(cfg: RunConfig, d: int) -> int:
    """INIT_RESPONSE payload bytes (transport.py:391-396)."""
    size = 0
    if cfg.is_pp:
        size += 8 + 8 * d
    if cfg.hessian_init == "exact":
        size += 8 * packed_length(d)
    return size
