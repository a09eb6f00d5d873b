"""Sharding and collectives for multi-GPU search (one process per GPU).

* chains shard by rank: rank r owns seeds ``base + r*C .. base + r*C + C-1``
  (the reference's consecutive seeds, driver.py:73-79, split across ranks);
* every epoch the ranks all-gather one (energy, seed, rank) record each and
  adopt the minimum under the reference's ranking key (driver.py:81-85:
  best time, then seed); the owner broadcasts its schedule;
* verification shards samples by batch index and merges verdicts with
  sum(passed), sum(failed), min(first failing sample) (SPEC: deterministic merge).

Works with any torch.distributed backend: NCCL over NVLink on the B200 box
(tensors on the rank's GPU), gloo on CPU for the tests.
"""
from __future__ import annotations

import numpy as np


def shard_seeds(base: int, rank: int, chains: int, epoch: int = 0, world: int = 1) -> np.ndarray:
    return np.arange(chains, dtype=np.int64) + (epoch * world + rank) * chains + base


def exchange_best(dist, energy: float, seed: int, sched: np.ndarray, device=None):
    """All-gather (energy, seed, rank); return (best energy, best seed, owner, schedule)."""
    import torch

    rank, world = dist.get_rank(), dist.get_world_size()
    dev = device if device is not None else torch.device("cpu")
    mine = torch.tensor([float(energy), float(seed), float(rank)], dtype=torch.float64, device=dev)
    allv = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allv, mine)
    rows = sorted(tuple(float(x) for x in v.tolist()) for v in allv)
    e, s, owner = rows[0]
    buf = torch.as_tensor(np.asarray(sched, dtype=np.int32), device=dev).clone()
    dist.broadcast(buf, src=int(owner))
    return e, int(s), int(owner), buf.cpu().numpy().astype(np.uint16)


def merge_verdicts(dist, passed: int, failed: int, first_fail: int, device=None):
    """Sum passed/failed and take the minimum first failing sample over ranks (-1 = none)."""
    import torch

    dev = device if device is not None else torch.device("cpu")
    big = float(2 ** 62)
    t = torch.tensor([float(passed), float(failed)], dtype=torch.float64, device=dev)
    f = torch.tensor([float(first_fail) if first_fail >= 0 else big], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    dist.all_reduce(f, op=dist.ReduceOp.MIN)
    ff = int(f.item())
    return int(t[0].item()), int(t[1].item()), (-1 if ff >= big else ff)
