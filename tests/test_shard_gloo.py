"""Multi-rank (world_size 2, gloo, CPU) test of the guest-sharded scheduler.

Each rank builds the same scaled-down C5 world with this package's control
plane, translates the VA batches of the guests it owns, and returns the
results to rank 0 point-to-point; rank 0 must end up with exactly the
single-process results for every guest.  The per-guest "kernel" here is the
CPU oracle (no GPU on this box); on a GPU box the same scheduler runs the
CUDA walk (bench.py).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _world():
    import sys

    sys.path.insert(0, ROOT)
    from paper_1304_3771_b200 import workloads as W

    cfg = W.C5Config(guests=4, guest_bytes=8 << 20, host_private=16 << 20, procs=2, pages_per_proc=600,
                     vas_per_guest=5000, copy_bytes_per_guest=1 << 20, op_bytes=64 << 10)
    return cfg, W.build_c5(cfg)


def _guest_result(cfg, world, g):
    from oracle import oracle as O
    from paper_1304_3771_b200 import workloads as W

    img = world.memv.host_mem.backing.host
    vals, stats = [], []
    for p, vas in enumerate(W.c5_vas(cfg, g)):
        sp = O.space(0, world.spaces[g][p].shadow_root.root_pfn)
        v, s, _ = O.translate(img, sp, vas.astype(np.uint64), threads=1)
        vals.append(v.view(np.int64))
        stats.append(s.view(np.int32))
    return {"value": torch.from_numpy(np.concatenate(vals)), "status": torch.from_numpy(np.concatenate(stats))}


def _rank_main(rank, world_size, port, q):
    import sys

    sys.path.insert(0, ROOT)
    from paper_1304_3771_b200 import shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    try:
        cfg, world = _world()
        results = shard.run_owned(cfg.guests, rank, world_size, lambda g: _guest_result(cfg, world, g))
        n = cfg.vas_per_guest

        def like(g):
            return {"value": torch.empty(n, dtype=torch.int64), "status": torch.empty(n, dtype=torch.int32)}

        gathered = shard.gather_to_rank0(results, cfg.guests, rank, world_size, like)
        t = shard.max_over_ranks([float(rank + 1)], world_size)
        if rank == 0:
            q.put(({g: {k: v.numpy().copy() for k, v in r.items()} for g, r in gathered.items()}, t))
    finally:
        dist.destroy_process_group()


def test_owned_guests_partition():
    from paper_1304_3771_b200 import shard

    for world in (1, 2, 4, 8):
        seen = sorted(g for r in range(world) for g in shard.owned_guests(8, r, world))
        assert seen == list(range(8))
    assert shard.owned_guests(8, 1, 4) == [1, 5]
    with pytest.raises(ValueError):
        shard.owned_guests(8, 4, 4)


def test_two_rank_gloo_gather_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, t = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == [2.0]  # max over ranks
    cfg, world = _world()
    assert sorted(gathered) == list(range(cfg.guests))
    for g in range(cfg.guests):
        ref = _guest_result(cfg, world, g)
        assert np.array_equal(gathered[g]["value"], ref["value"].numpy())
        assert np.array_equal(gathered[g]["status"], ref["status"].numpy())
        assert (gathered[g]["status"] == 0).all()
