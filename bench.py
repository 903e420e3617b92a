"""Benchmark: FedNL rounds/s at d=301, n=142 on one B200 (BASELINE config c0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c0] [--impl ours|reference]

A "step" is one FedNL round (all n clients' oracle, Hessian-shift
compressor, fused shift + master fold, master Cholesky step) over the
config's synthetic shards (SURVEY §8(d) stand-ins for the W8A shape).

ours       value = K rounds / device time (CUDA events on the round stream,
           graph replays, shards resident in HBM); e2e = K rounds through the
           public `simulate(cfg, shards)` call from host shards (upload,
           init, rounds, rows back) ; roofline of the dominant kernel (the
           fp64 DMMA Hessian) against the in-repo fp64 peak; cpu_baseline =
           the numpy restatement of the reference (oracle/) on the host cores.
reference  the reference algorithm's CPU path (the oracle port; the reference
           is pure Python and not installed on the GPU box) on all host
           cores, one round per step; rank 0 only under torchrun.

N > 1 (torchrun): FedNL and FedNL-LS shard the clients over the ranks
(fb_set_shard: per-round NCCL all-gathers, every rank holds the identical
master state; "scaling": "strong", value = rounds / max-over-ranks device
time); FedNL-PP runs independent replicas (value = sum over ranks).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FedNL rounds/s at d=301,n=142 on 1 GPU; Hessian fp64 TFLOP/s and compressor GB/s"


def _env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ------------------------------------------------------------------ clocks


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region: an NVML thread polling every ~0.2 ms (a c0 run of 20 rounds lasts
    under 10 ms, below nvidia-smi's 10 ms period)."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples: list[tuple[float, int]] = []  # (sm MHz, reasons bitmask)
        self.smax = None
        self.stop = threading.Event()
        self.nv = None

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            self.smax = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
            self.bits = {
                "hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap,
            }
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001 - no NVML: no samples (reported as such)
            self.nv = None
        return self

    def _poll(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((float(sm), int(rs)))
            except Exception:  # noqa: BLE001
                return
            time.sleep(0.0002)

    def __exit__(self, *exc):
        self.stop.set()
        if self.nv is not None:
            self.t.join(timeout=2)

    def summary(self) -> dict:
        sm = sorted(v for v, _ in self.samples)
        reasons = set()
        for _, rs in self.samples:
            for nm in self.NAMES:
                if rs & self.bits[nm]:
                    reasons.add(nm)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": self.smax,
                "reasons": sorted(reasons), "samples": len(sm), "source": "NVML, ~0.2 ms period"}


# ------------------------------------------------------------------- peaks


def measured_peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            return json.load(fh)
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


# -------------------------------------------------------------- workloads


def build_inputs(config: str):
    from paper_2410_08760_b200 import data as D

    shards = D.baseline_shards(config, seed=1)
    return shards


def workload_label(config: str) -> str:
    """The workload string both arms print (the driver compares them)."""
    from paper_2410_08760_b200.data import BASELINE_CONFIGS

    c = BASELINE_CONFIGS[config]
    alg = {"fednl": "FedNL option b", "fednl-ls": "FedNL-LS option b (c=0.49, gamma=0.5)",
           "fednl-pp": f"FedNL-PP option b (tau={c.get('tau')})"}[c["algorithm"]]
    kind = {"topk": "TopK", "toplek": "TopLEK", "randk": "RandK", "randseqk": "RandSeqK"}[c["kind"]]
    alpha = "alpha=1" if c["alpha"] == 1.0 else "alpha default"
    gen = ("sparse-binary features" if c["gen"] == "binary" else "dense Gaussian features")
    return (f"{config}: {alg}, {kind} k={c['k']}, {alpha}, d={c['d']}, n={c['n']}, n_i={c['ni']}, "
            f"lambda={c['lam']:g}, {gen}")


def data_label(config: str) -> str:
    from paper_2410_08760_b200.data import BASELINE_CONFIGS

    c = BASELINE_CONFIGS[config]
    if c["gen"] == "binary":
        return "synthetic (SURVEY §8(d) sparse-binary stand-in for the paper's LIBSVM shape, seed 1)"
    return "synthetic (SURVEY §8(d) dense Gaussian stress input, numpy default_rng seed 1)"


def hessian_traffic(config: str):
    """ncu DRAM bytes per Hessian launch (dram__bytes_read.sum +
    dram__bytes_write.sum), from the committed capture of the current kernel."""
    tpath = os.path.join(ROOT, "profiles", "hessian_traffic.json")
    if not os.path.exists(tpath):
        return None, None
    with open(tpath) as fh:
        t = json.load(fh)
    e = t.get(config)
    if not isinstance(e, dict):
        return None, None
    return e.get("bytes_per_launch"), e.get("source")


def algorithmic_counts(config: str) -> dict:
    from paper_2410_08760_b200.data import BASELINE_CONFIGS

    c = BASELINE_CONFIGS[config]
    d, n, ni, k = c["d"], c["n"], c["ni"], c["k"]
    w = d * (d + 1) // 2
    n_act = c.get("tau", n) if c["algorithm"] == "fednl-pp" else n
    flops = n_act * ni * d * (d + 1)  # one FMA per (sample, packed entry)
    if c["kind"] in ("topk", "toplek"):
        comp_bytes = n_act * (8 * w + 12 * k)
    elif c["kind"] == "randseqk":
        comp_bytes = n_act * (16 * k + 8)
    else:
        comp_bytes = n_act * 20 * k
    # the shift update's random 8-byte read-modify-writes of H_i^k move whole
    # 32-byte sectors: (4 + 8) list bytes + a sector read and a sector written
    # per entry, the master's H^k once (contiguous)
    return {"hessian_flop": flops, "compress_bytes": comp_bytes, "fold_bytes": n_act * k * 44,
            "fold_sector_bytes": n_act * k * (12 + 64) + 16 * w,
            "oracle_bytes": n * d * ni * 8 * 2, "d": d, "n": n, "ni": ni, "k": k, "w": w}


# --------------------------------------------------------------- our arm


def run_ours(args) -> dict | None:
    import numpy as np

    import __graft_entry__ as G

    G.build()
    from paper_2410_08760_b200 import _lib, simulate
    from paper_2410_08760_b200.data import baseline_run_config
    from paper_2410_08760_b200.engine import FedNLEngine, fp64_peak

    rank, world, local = _env_rank()
    if world > 1:
        os.environ.setdefault("CUDA_VISIBLE_DEVICES", str(local))
    info = _lib.device_info()
    K, W = args.steps, args.warmup
    shards = build_inputs(args.config)
    cfg = baseline_run_config(args.config, rounds=K)
    d, n, ni = shards[0].dim, len(shards), shards[0].n_samples
    counts = algorithmic_counts(args.config)

    # ---- multi-GPU (torchrun): FedNL / FedNL-LS shard the clients over the
    # ranks (fb_set_shard: per-round NCCL all-gathers, bit-identical master
    # state on every rank); FedNL-PP runs independent replicas
    dist = None
    sharded = world > 1 and cfg.algorithm in ("fednl", "fednl-ls")
    nccl_id = None
    if world > 1:
        import torch
        import torch.distributed as dist

        dist.init_process_group("gloo")
        if sharded:
            from paper_2410_08760_b200.engine import nccl_unique_id

            box = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(box, src=0)
            nccl_id = box[0]

    def make_engine():
        e = FedNLEngine(cfg, d, n, ni, topk_path=args.topk_path)
        if sharded:
            e.set_shard(world, rank, nccl_id)
        return e

    # ---- device-resident throughput (value) + per-kernel CUDA events
    eng = make_engine()
    eng.upload([s.bmat for s in shards], [s.lam for s in shards])
    eng.init_state()
    eng.run_rounds(W)  # warm-up: graph capture, caches, clocks
    if dist is not None:
        dist.barrier()
    # timed region: the production round graph (CUDA events only at round
    # boundaries: a per-kernel event-record node between two kernels costs
    # their launch overlap, 24 us per c0 round)
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        batch = eng.run_rounds(K)
        wall = time.perf_counter() - t0
    dev_ms = float(batch.wall_ms[-1])  # device time of the K rounds (events)
    # per-kernel CUDA events (roofline, kernels_ms): the same rounds with the
    # event-instrumented graph, right after the timed region
    inst = eng.run_rounds(K, timed=True)
    inst_ms = float(inst.wall_ms[-1])
    prof = eng.profile()
    eng.close()

    # ---- multi-rank: max device time over ranks
    if dist is not None:
        t = torch.tensor([dev_ms, inst_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms, inst_ms = float(t[0].item()), float(t[1].item())
        dist.barrier()
    jobs = 1 if sharded else world  # replicas each run the whole job
    value = jobs * K / (dev_ms * 1e-3)

    # ---- end to end through the public API from host shards
    cfg_e2e = baseline_run_config(args.config, rounds=K)
    if sharded:  # the sharded engine from host shards: upload, init, K rounds, rows back
        t0 = time.perf_counter()
        e2 = make_engine()
        e2.upload([s.bmat for s in shards], [s.lam for s in shards])
        e2.init_state()
        rows = e2.run_rounds(K)
        e2.close()
        e2e_s = time.perf_counter() - t0
        t = torch.tensor([e2e_s], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
        final_gn = float(rows.grad_norm[-1])
    else:
        t0 = time.perf_counter()
        rows = simulate(cfg_e2e, shards)
        e2e_s = time.perf_counter() - t0
        final_gn = rows[-1].grad_norm
        if dist is not None:
            t = torch.tensor([e2e_s], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
    shard_bytes = sum(s.bmat.nbytes for s in shards) // (world if sharded else 1)
    row_bytes = (8 + 8 + 4 + 4 * n + 8)  # grad, f, ls, counts, wall per round

    if rank != 0:
        return None

    # ---- roofline of the dominant kernel (fp64 DMMA Hessian)
    dmma_peak, dfma_peak = fp64_peak()
    hess_ms = prof["ms_hessian"]
    achieved = counts["hessian_flop"] / (hess_ms * 1e-3) / 1e12
    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    comp_gbs = counts["compress_bytes"] / (prof["ms_compress"] * 1e-3) / 1e9 if prof["ms_compress"] else None
    fold_gbs = counts["fold_bytes"] / (prof["ms_fold"] * 1e-3) / 1e9 if prof["ms_fold"] else None
    fold_sec_gbs = counts["fold_sector_bytes"] / (prof["ms_fold"] * 1e-3) / 1e9 if prof["ms_fold"] else None
    traffic, traffic_src = hessian_traffic(args.config)

    cpu = None if args.no_cpu_baseline else cpu_baseline(args.config, budget_s=args.cpu_seconds)

    return {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "rounds/s",
        "n_gpus": world,
        "steps": K,
        "warmup": W,
        "ms_per_step": round(dev_ms / K, 5),
        "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": data_label(args.config),
        "config": {
            "workload": workload_label(args.config),
            "rounds_per_step": 1,
            "l2": (f"inputs larger than L2: per-round working set B {n * d * ni * 8 / 1e6:.1f} MB + "
                   f"H_i^k {n * counts['w'] * 8 / 1e6:.1f} MB + D {n * counts['w'] * 8 / 1e6:.1f} MB > 126 MB"),
            "parallelism": ("single GPU" if world == 1 else
                            f"clients sharded over {world} GPUs (NCCL all-gathers per round)" if sharded
                            else f"{world} independent replicas"),
        },
        "e2e": {
            "value": round(K / e2e_s, 3),
            "unit": "rounds/s",
            "h2d_bytes_per_step": int(shard_bytes // K),
            "d2h_bytes_per_step": row_bytes,
            "what": (f"sharded engine from host shards for {K} rounds incl. upload, init, rows (max over ranks)"
                     if sharded else f"simulate(cfg, shards) wall clock for {K} rounds incl. shard upload, init, rows"),
        },
        "gpu_launches": int(prof["launches_per_round"]) * K,
        "roofline": {
            "kernel": "k_hessian_ws (fp64 DMMA.8x8x4 SYRK + shift-difference epilogue)",
            "bound": "tensor",
            "achieved": round(achieved, 3),
            "peak": round(dmma_peak, 3),
            "unit": "TFLOP/s",
            "frac": round(achieved / dmma_peak, 4),
            "traffic": traffic,
            "traffic_unit": "bytes per launch",
            "traffic_source": traffic_src,
            "peak_source": "in-repo fp64 DMMA microbenchmark (MEASURED_PEAKS.json has no fp64 entry)",
            "algorithmic_flop_per_launch": counts["hessian_flop"],
            "ms_per_launch": round(hess_ms, 5),
            "timing": (f"CUDA events around k_hessian_ws on the round stream, {K} rounds of the "
                       "event-instrumented round graph run right after the timed region"),
        },
        "kernels_ms": {k[3:]: round(v, 5) for k, v in prof.items() if k.startswith("ms_")},
        "memory_kernels": {
            "compress_gbs": None if comp_gbs is None else round(comp_gbs, 1),
            "compress_frac_hbm": None if comp_gbs is None else round(comp_gbs / hbm, 4),
            "fold_gbs": None if fold_gbs is None else round(fold_gbs, 1),
            "fold_frac_hbm": None if fold_gbs is None else round(fold_gbs / hbm, 4),
            "fold_sector_gbs": None if fold_sec_gbs is None else round(fold_sec_gbs, 1),
            "fold_sector_frac_hbm": None if fold_sec_gbs is None else round(fold_sec_gbs / hbm, 4),
            "hbm_peak_gbs": hbm,
        },
        "fp64_peaks_tflops": {"dmma": round(dmma_peak, 2), "dfma": round(dfma_peak, 2)},
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "device": info["name"],
        "host_wall_s": round(wall, 4),
        "value_with_kernel_events": round(jobs * K / (inst_ms * 1e-3), 3),
        "final_grad_norm_e2e": final_gn,
    }


# ------------------------------------------------------ CPU (oracle port)


def _limit_blas_threads() -> None:
    """One BLAS thread per worker: threadpoolctl only limits libraries that are
    already loaded, so numpy is imported first."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import numpy  # noqa: F401

    try:
        import threadpoolctl

        threadpoolctl.threadpool_limits(1, "blas")
    except ImportError:
        pass


def _cpu_run(config: str, workers: int):
    from oracle import fednl_oracle as O
    from paper_2410_08760_b200.data import baseline_run_config

    shards = build_inputs(config)
    cfg = O.OracleConfig.from_run_config(baseline_run_config(config, rounds=10**6))
    run = O.OracleRun(cfg, [s.bmat for s in shards], lam=[s.lam for s in shards], workers=workers)
    run.init()
    return run


def _cpu_round(run, r: int) -> None:
    if run.cfg.algorithm == "fednl-pp":
        run.pp_round(r)
    else:
        run.fednl_round(r)


def cpu_baseline(config: str, budget_s: float = 12.0) -> dict:
    """The oracle port (oracle/, pinned to the reference's own rows) on the
    host cores: rounds run until `budget_s` of CPU time has elapsed (at least
    4), after one warm-up round."""
    _limit_blas_threads()
    workers = os.cpu_count() or 1
    run = _cpu_run(config, workers)
    try:
        _cpu_round(run, 0)
        t0 = time.perf_counter()
        r = 1
        while r < 5 or time.perf_counter() - t0 < budget_s:
            _cpu_round(run, r)
            r += 1
        dt = time.perf_counter() - t0
    finally:
        run.close()
    rounds = r - 1
    return {"value": round(rounds / dt, 4), "unit": "rounds/s", "cores": workers, "kind": "port",
            "sample": f"{rounds} rounds of {config} ({dt:.1f} s) after 1 warm-up round: numpy oracle port, "
                      f"{workers} worker threads, OpenBLAS 1 thread each"}


def run_reference(args) -> dict | None:
    rank, world, _ = _env_rank()
    if rank != 0:
        return None
    _limit_blas_threads()
    workers = os.cpu_count() or 1
    K, W = args.steps, args.warmup
    run = _cpu_run(args.config, workers)
    try:
        for r in range(W):
            _cpu_round(run, r)
        t0 = time.perf_counter()
        for r in range(W, W + K):
            _cpu_round(run, r)
        dt = time.perf_counter() - t0
    finally:
        run.close()
    v = K / dt
    return {
        "metric": METRIC, "value": round(v, 4), "unit": "rounds/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": round(1e3 * dt / K, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": data_label(args.config),
        "config": {"workload": workload_label(args.config),
                   "rounds_per_step": 1, "parallelism": f"CPU, {workers} threads"},
        "impl": "reference",
        "cpu_baseline": {"value": round(v, 4), "unit": "rounds/s", "cores": workers, "kind": "port",
                         "sample": f"{K} rounds after {W} warm-up rounds, numpy restatement of the "
                                   f"reference path (oracle/fednl_oracle.py), {workers} worker threads"},
        "e2e": {"value": round(v, 4), "unit": "rounds/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c0")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--topk-path", type=int, default=0, help=argparse.SUPPRESS)  # A/B of TopK variants
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    out = run_reference(args) if args.impl == "reference" else run_ours(args)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
