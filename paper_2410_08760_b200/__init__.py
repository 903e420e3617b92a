"""B200-native simulated FedNL round (arxiv/paper_2410_08760).

Drop-in for the reference package `fednl` on its hot path: the public names
of reference pkg/src/fednl/__init__.py:10-47 that concern the simulator are
re-exported with the same semantics; the arithmetic runs in hand-written
sm_100a CUDA (libfednl_b200.so) reached through a ctypes C ABI
(include/fednl_b200.h).  There is no CPU fallback.
"""

from .config import (
    CompressedDelta,
    CompressorKind,
    CompressorSpec,
    DivergenceError,
    EigenConvergenceError,
    LineSearchError,
    NotPositiveDefiniteError,
    RunConfig,
    StepInfo,
    default_alpha,
    resolve_alpha,
)
from .data import ClientShard
from .runtime import (
    MetricsRow,
    canonical_config,
    read_csv,
    run_client,
    run_master,
    simulate,
    traffic_model,
    write_csv,
)

__version__ = "0.1.0"

__all__ = [
    "ClientShard",
    "CompressedDelta",
    "CompressorKind",
    "CompressorSpec",
    "DivergenceError",
    "EigenConvergenceError",
    "LineSearchError",
    "MetricsRow",
    "NotPositiveDefiniteError",
    "RunConfig",
    "StepInfo",
    "canonical_config",
    "default_alpha",
    "read_csv",
    "resolve_alpha",
    "run_client",
    "run_master",
    "simulate",
    "traffic_model",
    "write_csv",
    "__version__",
]
