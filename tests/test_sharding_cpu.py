"""Client sharding across ranks, checked on CPU with gloo.

The library's multi-GPU path (fb_set_shard) gives each rank the clients
`shard_range(n, world, rank)`, all-gathers every client's round outputs
(gradient, loss / Frobenius partials, compressed delta) and runs the same
ascending-client reduction, master solve and fold on every rank.  This test
replays that decomposition with the CPU oracle on world_size 2 (gloo,
127.0.0.1): each rank evaluates only its own clients, the per-client results
are all-gathered, and both ranks must reproduce the single-process
trajectory bit for bit (and agree with each other).  An odd client count
exercises the padded last block.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.timeout(300)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(n=5, d=17, ni=24, seed=3):
    rng = np.random.default_rng(seed)
    bmats = []
    for _ in range(n):
        feats = (rng.random((d - 1, ni)) < 0.3).astype(np.float64)
        y = np.where(rng.random(ni) < 0.4, 1.0, -1.0)
        bmats.append(np.asfortranarray(np.vstack([feats, np.ones((1, ni))]) * y))
    return bmats


def _worker(rank: int, world: int, port: int, rounds: int, out_q) -> None:
    import torch.distributed as dist

    from oracle import fednl_oracle as O
    from paper_2410_08760_b200.engine import shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bmats = _problem()
        n, d = len(bmats), bmats[0].shape[0]
        cfg = O.OracleConfig(algorithm="fednl", kind="topk", k=2 * d, rounds=rounds, alpha=1.0, lam=1e-3,
                             run_seed=7)
        lo, hi = shard_range(n, world, rank)

        class ShardedRun(O.OracleRun):
            """Client work only for [lo, hi); results all-gathered in client order."""

            def _map(self, fn, cids):
                mine = {c: fn(c) for c in cids if lo <= c < hi}
                parts = [None] * world
                dist.all_gather_object(parts, mine)
                merged = {}
                for p in parts:
                    merged.update(p)
                assert sorted(merged) == list(cids)
                return merged

        ref = O.OracleRun(cfg, bmats, lam=1e-3)
        run = ShardedRun(cfg, bmats, lam=1e-3)
        ref.init()
        run.init()
        ref_rows, rows = [], []
        for r in range(rounds):
            ref_rows.append(ref.fednl_round(r))
            rows.append(run.fednl_round(r))
        ok = (np.array_equal(ref.x, run.x) and np.array_equal(ref.h_mas, run.h_mas) and
              all(a.grad_norm == b.grad_norm and a.f_value == b.f_value for a, b in zip(ref_rows, rows)))
        xs = [None] * world
        dist.all_gather_object(xs, run.x.tolist())
        same = all(x == xs[0] for x in xs)
        out_q.put((rank, ok, same, (lo, hi)))
    finally:
        dist.destroy_process_group()


def test_two_rank_client_sharding_reproduces_single_process_rounds():
    import torch.multiprocessing as mp

    world, rounds = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, rounds, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    res.sort()
    ranges = [r[3] for r in res]
    assert ranges == [(0, 3), (3, 5)]  # ceil(5 / 2) = 3 clients per block
    for rank, ok, same, _ in res:
        assert ok, f"rank {rank} diverged from the single-process oracle"
        assert same, f"rank {rank} disagrees with the other ranks"


def test_shard_range_partitions_every_client_once():
    from paper_2410_08760_b200.engine import shard_range

    for n in (1, 5, 142, 512):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                lo, hi = shard_range(n, world, r)
                assert 0 <= lo <= hi <= n
                seen.extend(range(lo, hi))
            assert seen == list(range(n))
