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


def _worker_ls_pp(rank: int, world: int, port: int, out_q) -> None:
    """FedNL-LS (trial losses per client, all-gathered per trial batch) and
    FedNL-PP (participant slots split over the ranks, per-slot outputs
    exchanged, the non-owners applying the client update) — the
    decompositions fb_set_shard runs on the GPUs, replayed with the oracle."""
    import torch.distributed as dist

    from oracle import fednl_oracle as O
    from paper_2410_08760_b200.engine import shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bmats = _problem()
        n, d = len(bmats), bmats[0].shape[0]
        lo, hi = shard_range(n, world, rank)
        results = {}

        # ---- FedNL-LS: every client-map (round work and the trial f) sharded by client
        class ShardedLS(O.OracleRun):
            def _map(self, fn, cids):
                mine = {c: fn(c) for c in cids if lo <= c < hi}
                parts = [None] * world
                dist.all_gather_object(parts, mine)
                merged = {}
                for p in parts:
                    merged.update(p)
                return merged

        cfg = O.OracleConfig(algorithm="fednl-ls", kind="topk", k=2 * d, rounds=4, ls_c=0.99, ls_gamma=0.8,
                             lam=1e-3, run_seed=5)
        ref, run = O.OracleRun(cfg, bmats, lam=1e-3), ShardedLS(cfg, bmats, lam=1e-3)
        ref_rows, rows = ref.run(), run.run()
        results["ls"] = (np.array_equal(ref.x, run.x) and
                         [(r.grad_norm, r.ls_steps) for r in ref_rows] == [(r.grad_norm, r.ls_steps) for r in rows]
                         and max(r.ls_steps for r in rows) >= 4)

        # ---- FedNL-PP: participant slots [r * spr, (r + 1) * spr) per rank
        class ShardedPP(O.OracleRun):
            def _map(self, fn, cids):
                if fn.__name__ != "<lambda>" or len(cids) == self.n:  # probes: by client range
                    mine = {c: fn(c) for c in cids if lo <= c < hi}
                    parts = [None] * world
                    dist.all_gather_object(parts, mine)
                    merged = {}
                    for p in parts:
                        merged.update(p)
                    return merged
                spr = (len(cids) + world - 1) // world
                mine_slots = cids[rank * spr:(rank + 1) * spr]
                mine = {}
                for c in mine_slots:
                    res = fn(c)  # the owner applies its client's update itself
                    mine[c] = (res, self.h_cli[c].copy(), self.cli_shift[c], self.cli_gvec[c].copy())
                parts = [None] * world
                dist.all_gather_object(parts, mine)
                merged = {}
                for p in parts:
                    for c, (res, h, sh, gv) in p.items():
                        if c not in mine:  # a non-owner: the owner's client state
                            self.h_cli[c] = h
                            self.cli_shift[c] = sh
                            self.cli_gvec[c] = gv
                        merged[c] = res
                return merged

        cfg = O.OracleConfig(algorithm="fednl-pp", kind="randk", k=d, rounds=6, tau=3, lam=1e-3, run_seed=9)
        ref, run = O.OracleRun(cfg, bmats, lam=1e-3), ShardedPP(cfg, bmats, lam=1e-3)
        ref_rows, rows = ref.run(), run.run()
        results["pp"] = (np.array_equal(ref.x, run.x) and np.array_equal(ref.h_cli, run.h_cli) and
                         [r.grad_norm for r in ref_rows] == [r.grad_norm for r in rows])
        out_q.put((rank, results))
    finally:
        dist.destroy_process_group()


def test_two_rank_ls_and_pp_sharding_reproduce_single_process_rounds():
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_ls_pp, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, r in sorted(res):
        assert r["ls"], f"rank {rank}: sharded FedNL-LS diverged"
        assert r["pp"], f"rank {rank}: sharded FedNL-PP diverged"
