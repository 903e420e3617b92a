"""`simulate(cfg, shards)` — the drop-in simulator entry point.

Same signature, contract and MetricsRow output as the reference's
runtime.simulate (runtime.py:136-276): R rows (one per executed round,
describing the iterate entering it and the cumulative traffic through its
exchange) plus a final evaluation row, byte counters equal to the
reference's wire accounting, `workers` accepted and ignored (all clients run
on the GPU; no output depends on it).  The arithmetic runs in
libfednl_b200.so; this module only shapes inputs and rows.
"""

from __future__ import annotations

import time
from dataclasses import dataclass
from typing import IO, Iterable

import numpy as np

from .config import (
    CompressorKind,
    RunConfig,
    init_response_size,
    packed_length,
    resolve_alpha,
    update_payload_size,
    wire_size_bytes,
)
from .data import ClientShard
from .engine import FedNLEngine

CSV_HEADER = "round,wall_seconds,grad_norm,f_value,bytes_up_cum,bytes_down_cum,ls_steps"


@dataclass
class MetricsRow:
    """runtime.py:54-62."""

    round: int
    wall_seconds: float
    grad_norm: float
    f_value: float
    bytes_up_cum: int
    bytes_down_cum: int
    ls_steps: int


def _g17(v: float) -> str:
    return "%.17g" % v


def write_csv(rows: Iterable[MetricsRow], dest: str | IO[str], config_line: str | None = None) -> None:
    """runtime.py:69-86: '# config:' comment, header, %.17g floats."""
    own = isinstance(dest, str)
    fh = open(dest, "w") if own else dest
    try:
        if config_line is not None:
            fh.write(f"# config: {config_line}\n")
        fh.write(CSV_HEADER + "\n")
        for r in rows:
            fh.write(
                f"{r.round},{_g17(r.wall_seconds)},{_g17(r.grad_norm)},"
                f"{_g17(r.f_value)},{r.bytes_up_cum},{r.bytes_down_cum},{r.ls_steps}\n"
            )
    finally:
        if own:
            fh.close()


def read_csv(path: str) -> tuple[str | None, list[MetricsRow]]:
    """runtime.py:89-113."""
    config_line = None
    rows: list[MetricsRow] = []
    with open(path) as fh:
        for line in fh:
            line = line.rstrip("\n")
            if line.startswith("# config: "):
                config_line = line[len("# config: "):]
                continue
            if not line or line == CSV_HEADER:
                continue
            c = line.split(",")
            rows.append(MetricsRow(int(c[0]), float(c[1]), float(c[2]), float(c[3]),
                                   int(c[4]), int(c[5]), int(c[6])))
    return config_line, rows


def canonical_config(cfg: RunConfig, d: int, n_clients: int) -> str:
    """transport.py:205-232: the one-line run identity echoed in CSVs."""
    w = packed_length(d)
    comp = cfg.compressor
    pairs = [
        ("algorithm", cfg.algorithm),
        ("option", cfg.option),
        ("compressor", comp.kind.value),
        ("k", str(comp.k) if comp.k is not None else "-"),
        ("topk-ranking", "weighted" if comp.topk_weighted else "raw"),
        ("alpha", repr(resolve_alpha(cfg, w))),
        ("lambda", repr(cfg.lam)),
        ("mu", repr(cfg.effective_mu)),
        ("c", repr(cfg.ls_c)),
        ("gamma", repr(cfg.ls_gamma)),
        ("tau", str(cfg.tau) if cfg.tau is not None else "-"),
        ("rounds", str(cfg.rounds)),
        ("seed", str(cfg.run_seed)),
        ("hessian-init", cfg.hessian_init),
        ("reconstruct-indices", "on" if cfg.reconstruct_indices else "off"),
        ("d", str(d)),
        ("clients", str(n_clients)),
    ]
    return " ".join(f"{k}={v}" for k, v in pairs)


@dataclass
class TrafficModel:
    """runtime.py:279-294."""

    delta_bytes: int
    update_bytes: int
    total_up_bytes: int
    total_down_bytes: int

    @property
    def up_mib(self) -> float:
        return self.total_up_bytes / 2.0**20

    @property
    def down_mib(self) -> float:
        return self.total_down_bytes / 2.0**20


def model_delta_bytes(cfg: RunConfig, d: int) -> int:
    """runtime.py:297-317."""
    w = packed_length(d)
    kind = cfg.compressor.kind
    cfg.compressor.validate(w)
    if kind is CompressorKind.IDENTITY:
        return 8 * w
    if kind is CompressorKind.NATURAL:
        return (12 * w + 7) // 8
    if kind in (CompressorKind.RANDK, CompressorKind.RANDSEQK):
        return 8 + 8 * cfg.compressor.k if cfg.reconstruct_indices else 12 * cfg.compressor.k
    return 12 * cfg.compressor.k


def traffic_model(cfg: RunConfig, d: int, n_clients: int, rounds: int) -> TrafficModel:
    """runtime.py:320-330."""
    delta = model_delta_bytes(cfg, d)
    update = update_payload_size(cfg, d, delta)
    return TrafficModel(delta, update, rounds * n_clients * update, rounds * n_clients * 8 * d)


def _validate(cfg: RunConfig, shards: list[ClientShard]) -> tuple[int, int, int]:
    n = len(shards)
    if n == 0:
        raise ValueError("need at least one shard")
    d = shards[0].dim
    if any(s.dim != d for s in shards):
        raise ValueError("all shards must share one dimension")
    cfg.validate(n)
    ni = max(s.n_samples for s in shards)  # shards may be ragged (runtime.py:145-151)
    packed_length(d)
    cfg.compressor.validate(packed_length(d))
    return n, d, ni


def _update_bytes(cfg: RunConfig, d: int, kind: CompressorKind, counts: np.ndarray) -> np.ndarray:
    """Sum over participants (count >= 0; PP marks absent clients -1) of the
    CLIENT_UPDATE payload per round: update_payload_size(wire_size_bytes(count))
    (transport.py:383-388, compressors.py:465-482), vectorised."""
    c = counts.astype(np.int64)
    part = c >= 0
    w = packed_length(d)
    if kind is CompressorKind.IDENTITY:
        wire = np.full_like(c, 8 * w)
    elif kind is CompressorKind.NATURAL:
        wire = np.full_like(c, (12 * w + 7) // 8)
    elif kind in (CompressorKind.RANDK, CompressorKind.RANDSEQK) and cfg.reconstruct_indices:
        wire = 8 + 8 * c
    else:
        wire = 12 * c
    wire = np.where(c == 0, 0, wire)
    base = update_payload_size(cfg, d, 0)
    return np.where(part, base + wire, 0).sum(axis=1)


def simulate(cfg: RunConfig, shards: list[ClientShard], workers: int = 1,
             engine: FedNLEngine | None = None) -> list[MetricsRow]:
    """Single-process run over in-memory shards, every client on the GPU.

    `workers` is accepted for signature compatibility and ignored: the
    trajectory and counters never depended on it (runtime.py:141-143).
    Shards may differ in n_samples and lam: each client's oracle uses its
    shard's own (oracle.py:95-139), as the reference does.
    """
    del workers
    n, d, ni = _validate(cfg, shards)
    t0 = time.perf_counter()
    own = engine is None
    eng = engine or FedNLEngine(cfg, d, n, ni)
    try:
        eng.upload([s.bmat for s in shards], [s.lam for s in shards])
        eng.init_state()
        t_init = time.perf_counter() - t0
        up = down = 0
        if cfg.needs_init_exchange(n):  # runtime.py:226-228
            down += 8 * d * n
            up += n * init_response_size(cfg, d)
        batch = eng.run_rounds(cfg.rounds, stop_grad_norm=cfg.stop_grad_norm)
        rows: list[MetricsRow] = []
        kind = cfg.compressor.kind
        stopped = False
        # per-round uplink bytes of all participants, vectorised over clients
        up_round = _update_bytes(cfg, d, kind, batch.entry_counts[: batch.done])
        n_part = (batch.entry_counts[: batch.done] >= 0).sum(axis=1)
        for i in range(batch.done):
            n_i = int(n_part[i]) if cfg.is_pp else n
            gn = float(batch.grad_norm[i])
            if cfg.is_pp and cfg.stop_grad_norm is not None and gn <= cfg.stop_grad_norm:
                # runtime.py:239-242: the probe row is recorded before any traffic
                rows.append(MetricsRow(i, t_init + batch.wall_ms[i] * 1e-3, gn, float(batch.f_value[i]),
                                       up, down, 0))
                stopped = True
                break
            down += 8 * d * n_i
            up += int(up_round[i])
            if cfg.is_ls:  # runtime.py:203-208: every trial is traffic
                trials = int(batch.ls_steps[i]) + 1
                down += 8 * d * n * trials
                up += 8 * n * trials
            rows.append(MetricsRow(i, t_init + batch.wall_ms[i] * 1e-3, gn, float(batch.f_value[i]),
                                   up, down, int(batch.ls_steps[i])))
            if (not cfg.is_pp) and cfg.stop_grad_norm is not None and gn <= cfg.stop_grad_norm:
                stopped = True
                break
        if not stopped:
            gn, fv = eng.final_eval()
            rows.append(MetricsRow(cfg.rounds, time.perf_counter() - t0, gn, fv, up, down, 0))
        return rows
    finally:
        if own:
            eng.close()


def run_master(*args, **kwargs):  # pragma: no cover - out of scope
    raise NotImplementedError("the TCP master is outside this GPU build's scope; use simulate()")


def run_client(*args, **kwargs):  # pragma: no cover - out of scope
    raise NotImplementedError("the TCP client is outside this GPU build's scope; use simulate()")
