"""World-2 client sharding over NCCL (fb_set_shard), one process per GPU.

Runs only where two GPUs are visible (skipped otherwise: the build and
round-end boxes have one).  Each rank owns half of the clients (FedNL /
FedNL-LS) or half of each round's participant slots (FedNL-PP); every rank
must reproduce the single-GPU rows and iterate bit for bit.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _n_gpus() -> int:
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        return 0


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank: int, world: int, port: int, name: str, q) -> None:
    os.environ["CUDA_VISIBLE_DEVICES"] = str(rank)
    import torch.distributed as dist

    from cases_r2 import SIM_R2, case_r2, run_config
    from test_gpu_parity import SIM, sim_case
    from paper_2410_08760_b200 import simulate
    from paper_2410_08760_b200.engine import FedNLEngine, nccl_unique_id

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if name in SIM_R2:
            kw, shards = case_r2(name)
            cfg = run_config(kw)
        else:
            cfg, shards = sim_case(name)
        d, n, ni = shards[0].dim, len(shards), max(s.n_samples for s in shards)
        box = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        eng = FedNLEngine(cfg, d, n, ni)
        eng.set_shard(world, rank, box[0])
        rows = simulate(cfg, shards, engine=eng)
        x = eng.get_x()
        eng.close()
        ref = FedNLEngine(cfg, d, n, ni)
        ref_rows = simulate(cfg, shards, engine=ref)
        x_ref = ref.get_x()
        ref.close()
        ok = ([(r.grad_norm, r.f_value, r.bytes_up_cum, r.ls_steps) for r in rows] ==
              [(r.grad_norm, r.f_value, r.bytes_up_cum, r.ls_steps) for r in ref_rows]
              and np.array_equal(x, x_ref))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(_n_gpus() < 2, reason="needs two visible GPUs (world-2 NCCL)")
@pytest.mark.parametrize("name", ["c0_r4", "ls_topk", "fednl_natural", "pp_randk", "ls_deep", "ragged_pp"])
def test_world2_sharded_matches_single_gpu(name):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
