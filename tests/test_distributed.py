"""World-size-2 gloo tests of the multi-GPU plumbing (runs on CPU)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_16863_b200.parallel import (RED_MAX, TorchGroup, exchange_best, merge_verdicts,
                                            pick_winner, shard_seeds)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank 1 holds the better energy; ties would break by seed
        energy = [0.97, 0.95][rank]
        sched = np.arange(10, dtype=np.uint16)[::-1] if rank == 1 else np.arange(10, dtype=np.uint16)
        e, s, owner, got = exchange_best(dist, energy, 100 + rank, sched)
        # tie on energy: the smaller seed wins (driver.py:81-85 ranking)
        e2, s2, owner2, _ = exchange_best(dist, 0.9, 7 - rank, sched)
        g = TorchGroup(dist)
        p, f, ff = merge_verdicts(g, 1000 + rank, rank, 5000 if rank else -1)
        # the group interface the bench and HardwareSearch use
        ge, gs, gowner, ggot = g.exchange_best([0.97, 0.95][rank], 100 + rank, sched)
        assert (ge, gs, gowner) == (0.95, 101, 1) and ggot.tolist() == list(range(10))[::-1]
        assert g.allreduce([rank + 1.5], RED_MAX) == [2.5]
        assert g.broadcast_perm(sched, root=1).tolist() == list(range(10))[::-1]
        seeds = shard_seeds(0, rank, 4, epoch=1, world=world).tolist()
        q.put((rank, e, s, owner, got.tolist(), s2, owner2, p, f, ff, seeds))
    finally:
        dist.destroy_process_group()


def test_exchange_and_merge_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, e, s, owner, got, s2, owner2, p, f, ff, seeds in res:
        assert (e, s, owner) == (0.95, 101, 1)
        assert got == list(range(10))[::-1]
        assert (s2, owner2) == (6, 1)
        assert (p, f, ff) == (2001, 1, 5000)
        assert seeds == [8 + 4 * rank + i for i in range(4)]


def test_pick_winner_ranking_key():
    """driver.py:81-85: best time first, then seed; rank only breaks exact duplicates."""
    assert pick_winner([(0.9, 5, 0), (0.8, 9, 1)]) == (0.8, 9, 1)
    assert pick_winner([(0.9, 5, 0), (0.9, 3, 1)]) == (0.9, 3, 1)
    assert pick_winner([(0.9, 3, 1), (0.9, 3, 0)]) == (0.9, 3, 0)


@pytest.mark.gpu
def test_nccl_group_c_abi_single_rank():
    """libsip's NCCL communicator (sip_comm_* / sip_nccl_exchange) on one B200: a
    one-rank group exchanges with itself (the 8-GPU path is the same calls)."""
    from paper_2403_16863_b200.engine import get_context
    from paper_2403_16863_b200.parallel import RED_MAX, RED_SUM, NcclGroup

    g = NcclGroup(get_context(0), 0, 1)
    try:
        sched = np.arange(1184, dtype=np.uint16)[::-1].copy()
        e, s, owner, got = g.exchange_best(0.97, 42, sched)
        assert (e, s, owner) == (0.97, 42, 0) and np.array_equal(got, sched)
        assert g.allreduce([1.5, -2.0], RED_SUM) == [1.5, -2.0]
        assert g.allreduce([3.0], RED_MAX) == [3.0]
        assert np.array_equal(g.broadcast_perm(sched, 0), sched)
        g.barrier()
    finally:
        g.close()
