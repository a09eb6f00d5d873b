"""Sharding and collectives for multi-GPU search (one process per GPU).

* chains shard by rank: rank r owns seeds ``base + r*C .. base + r*C + C-1``
  (the reference's consecutive seeds, driver.py:73-79, split across ranks);
* every epoch the ranks all-gather one (energy, seed, rank) record each and
  adopt the minimum under the reference's ranking key (driver.py:81-85:
  best time, then seed); the owner broadcasts its schedule;
* verification shards samples by batch index and merges verdicts with
  sum(passed), sum(failed), min(first failing sample) (SPEC: deterministic merge).

Two implementations of the same group interface:

* :class:`NcclGroup` -- the product path: ``sip_comm_*`` / ``sip_nccl_exchange``
  in libsip (ncclAllGather of 24-byte records + ncclBroadcast of the winning
  schedule over NVLink).  torch.distributed is used only to hand rank 0's
  128-byte NCCL id to the other ranks (rendezvous, any backend).
* :class:`TorchGroup` -- the same interface over a torch.distributed process
  group, for the CPU (gloo) tests of the host logic and the one-GPU
  ``SIP_SHARE_DEVICE`` hook (NCCL refuses two ranks on one device).
"""
from __future__ import annotations

import ctypes

import numpy as np

RED_SUM, RED_MAX, RED_MIN = 0, 1, 2


class Best(ctypes.Structure):
    """sip_best (include/sip.h): one rank's epoch champion, 24 bytes."""
    _fields_ = [("energy", ctypes.c_double), ("seed", ctypes.c_int64), ("rank", ctypes.c_int32),
                ("pad", ctypes.c_int32)]


def shard_seeds(base: int, rank: int, chains: int, epoch: int = 0, world: int = 1) -> np.ndarray:
    return np.arange(chains, dtype=np.int64) + (epoch * world + rank) * chains + base


def pick_winner(records) -> tuple:
    """records: iterable of (energy, seed, rank) -> the one every rank adopts
    (driver.py:81-85 ranking: best time, then seed; rank breaks exact ties)."""
    return min((float(e), int(s), int(r)) for e, s, r in records)


class NcclGroup:
    """libsip's NCCL communicator (C ABI) for one rank."""

    def __init__(self, ctx, rank: int, world: int, rendezvous=None):
        """`rendezvous`: a torch.distributed module with an initialised process group
        (any backend) used once to broadcast rank 0's NCCL id."""
        from .engine import c_u8p

        self.ctx, self.rank, self.world = ctx, rank, world
        lib = ctx.lib
        uid = np.zeros(128, dtype=np.uint8)
        if rank == 0:
            rc = lib.sip_comm_unique_id(uid.ctypes.data_as(c_u8p))
            if rc != 0:
                raise RuntimeError("sip_comm_unique_id failed (libnccl.so.2 not loadable?)")
        if world > 1:
            if rendezvous is None:
                raise ValueError("world > 1 needs a rendezvous to share the NCCL id")
            box = [uid.tobytes()]
            rendezvous.broadcast_object_list(box, src=0)
            uid = np.frombuffer(box[0], dtype=np.uint8).copy()
        h = ctypes.c_void_p()
        ctx.check(lib.sip_comm_create(ctx.handle, uid.ctypes.data_as(c_u8p), world, rank, ctypes.byref(h)))
        self.handle = h

    def exchange_best(self, energy: float, seed: int, sched: np.ndarray):
        from .engine import c_u16p

        mine = Best(float(energy), int(seed), self.rank, 0)
        sched = np.ascontiguousarray(sched, dtype=np.uint16)
        out = np.zeros_like(sched)
        win = Best()
        allr = (Best * self.world)()
        self.ctx.check(self.ctx.lib.sip_nccl_exchange(
            self.handle, ctypes.byref(mine), sched.ctypes.data_as(c_u16p), len(sched), allr,
            ctypes.byref(win), out.ctypes.data_as(c_u16p)))
        return win.energy, int(win.seed), int(win.rank), out

    def allreduce(self, vals, op: int) -> list:
        from .engine import c_dblp

        v = np.ascontiguousarray(vals, dtype=np.float64).copy()
        self.ctx.check(self.ctx.lib.sip_comm_allreduce(self.handle, v.ctypes.data_as(c_dblp), len(v), op))
        return v.tolist()

    def broadcast_perm(self, perm: np.ndarray, root: int = 0) -> np.ndarray:
        """The root's schedule on every rank (an exchange whose only contender is root)."""
        e = float("-inf") if self.rank == root else float("inf")
        return self.exchange_best(e, 0, perm)[3]

    def barrier(self) -> None:
        self.ctx.check(self.ctx.lib.sip_comm_barrier(self.handle))

    def close(self) -> None:
        if self.handle:
            self.ctx.lib.sip_comm_destroy(self.handle)
            self.handle = None


class TorchGroup:
    """The group interface over torch.distributed (gloo on CPU in the tests)."""

    def __init__(self, dist, device=None):
        import torch

        self.dist = dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.device = device if device is not None else torch.device("cpu")

    def exchange_best(self, energy: float, seed: int, sched: np.ndarray):
        return exchange_best(self.dist, energy, seed, sched, self.device)

    def allreduce(self, vals, op: int) -> list:
        import torch

        t = torch.tensor(list(vals), dtype=torch.float64, device=self.device)
        red = {RED_SUM: self.dist.ReduceOp.SUM, RED_MAX: self.dist.ReduceOp.MAX,
               RED_MIN: self.dist.ReduceOp.MIN}[op]
        self.dist.all_reduce(t, op=red)
        return t.tolist()

    def broadcast_perm(self, perm: np.ndarray, root: int = 0) -> np.ndarray:
        import torch

        t = torch.as_tensor(np.asarray(perm, dtype=np.int32), device=self.device).clone()
        self.dist.broadcast(t, root)
        return t.cpu().numpy().astype(np.uint16)

    def barrier(self) -> None:
        self.dist.barrier()

    def close(self) -> None:
        pass


def exchange_best(dist, energy: float, seed: int, sched: np.ndarray, device=None):
    """All-gather (energy, seed, rank) over torch.distributed; return (best energy, best
    seed, owner, schedule)."""
    import torch

    rank, world = dist.get_rank(), dist.get_world_size()
    dev = device if device is not None else torch.device("cpu")
    mine = torch.tensor([float(energy), float(seed), float(rank)], dtype=torch.float64, device=dev)
    allv = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allv, mine)
    e, s, owner = pick_winner(tuple(v.tolist()) for v in allv)
    buf = torch.as_tensor(np.asarray(sched, dtype=np.int32), device=dev).clone()
    dist.broadcast(buf, src=int(owner))
    return e, int(s), int(owner), buf.cpu().numpy().astype(np.uint16)


def merge_verdicts(group, passed: int, failed: int, first_fail: int):
    """Sum passed/failed and take the minimum first failing sample over ranks (-1 = none)."""
    big = float(2 ** 62)
    p, f = group.allreduce([passed, failed], RED_SUM)
    ff = int(group.allreduce([first_fail if first_fail >= 0 else big], RED_MIN)[0])
    return int(p), int(f), (-1 if ff >= big else ff)
