"""Flatten a Kernel into the dense per-instruction tables the device consumes.

Layout (one entry per instruction *identity* = index in the input order):

``ctrl[i]`` (u32)   bits 0-5 wait mask, 6-8 read barrier (7 = none),
                    9-11 write barrier (7 = none), 12-16 issue advance
                    max(1, stall), 17-20 reuse bits (cubin listings only),
                    21 fence class (BARRIER/CONTROL_FLOW), 22 global class
``lat[i]``  (u32)   MachineConfig.latency_of (reference machine.py:76-85)
``klass[i]`` (u8)   ir.CLASS_CODE
``reads``/``writes`` u64[n*W] interned register bitsets (deps.reads_writes)
``refs``  (sip_memref[n*4]) memory references (deps.mem_refs)
``cut``   (u8[n+1]) 1 where a block boundary sits before position p
``pin``   (u8[n])   1 for instructions the hardware mode must never move
                    (EIATTR-listed offsets, relocation targets); 0 in parity mode

See include/sip.h for the C structs these arrays map onto.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .deps import mem_refs, reads_writes
from .ir import CLASS_CODE, GLOBAL_CLASSES, InstrClass, Kernel
from .machine import MachineConfig

MAX_REFS = 4
NO_BAR = 7
SPACE_CODE = {"global": 0, "shared": 1, "local": 2, "unknown": 3}


class MemRefC(ctypes.Structure):
    _fields_ = [
        ("offset", ctypes.c_int64),
        ("base", ctypes.c_int32),
        ("size", ctypes.c_uint8),
        ("space", ctypes.c_uint8),
        ("write", ctypes.c_uint8),
        ("pad", ctypes.c_uint8),
    ]


def pack_ctrl(ins, reuse: int = 0) -> int:
    c = ins.control
    if c is None:
        wait, rd, wr, adv = 0, NO_BAR, NO_BAR, 1
    else:
        wait = c.wait_bits
        rd = NO_BAR if c.read_barrier is None else c.read_barrier
        wr = NO_BAR if c.write_barrier is None else c.write_barrier
        adv = max(1, c.stall_cycles)
    fence = ins.klass in (InstrClass.BARRIER, InstrClass.CONTROL_FLOW)
    glob = ins.klass in GLOBAL_CLASSES
    return (wait | (rd << 6) | (wr << 9) | (adv << 12) | ((reuse & 0xF) << 17)
            | (int(fence) << 21) | (int(glob) << 22))


@dataclass
class KernelTables:
    n: int
    words: int
    ctrl: np.ndarray
    lat: np.ndarray
    klass: np.ndarray
    reads: np.ndarray
    writes: np.ndarray
    refs: np.ndarray          # structured view of MemRefC, shape (n*MAX_REFS,)
    nrefs: np.ndarray
    cut: np.ndarray
    pin: np.ndarray
    global_ids: np.ndarray    # identities of GLOBAL-class instructions, ascending
    names: tuple

    @classmethod
    def build(cls, kernel: Kernel, machine: MachineConfig | None = None,
              reuse=None, pinned=None) -> "KernelTables":
        cfg = machine or MachineConfig()
        sched = kernel.schedule
        n = len(sched)
        intern: dict = {}

        def rid(name: str) -> int:
            if name not in intern:
                intern[name] = len(intern)
            return intern[name]

        rw = [reads_writes(ins) for ins in sched]
        for r, w in rw:
            for name in sorted(r | w):
                rid(name)
        all_refs = [mem_refs(ins) for ins in sched]
        words = max(1, (len(intern) + 63) // 64)
        reads = np.zeros((n, words), dtype=np.uint64)
        writes = np.zeros((n, words), dtype=np.uint64)
        for i, (r, w) in enumerate(rw):
            for name in r:
                b = intern[name]
                reads[i, b >> 6] |= np.uint64(1 << (b & 63))
            for name in w:
                b = intern[name]
                writes[i, b >> 6] |= np.uint64(1 << (b & 63))

        refs = (MemRefC * (n * MAX_REFS))()
        nrefs = np.zeros(n, dtype=np.uint8)
        for i, lst in enumerate(all_refs):
            if len(lst) > MAX_REFS:
                raise ValueError(f"instruction {i} has {len(lst)} memory operands (max {MAX_REFS})")
            nrefs[i] = len(lst)
            for j, ref in enumerate(lst):
                slot = refs[i * MAX_REFS + j]
                slot.offset = int(ref.offset)
                slot.base = -1 if ref.base is None else rid(ref.base)
                slot.size = ref.size
                slot.space = SPACE_CODE[ref.space]
                slot.write = int(ref.write)

        reuse = reuse if reuse is not None else [0] * n
        ctrl = np.array([pack_ctrl(ins, reuse[i]) for i, ins in enumerate(sched)], dtype=np.uint32)
        lat = np.array([cfg.latency_of(ins) for ins in sched], dtype=np.uint32)
        klass = np.array([CLASS_CODE[ins.klass] for ins in sched], dtype=np.uint8)
        cut = np.zeros(n + 1, dtype=np.uint8)
        for p in kernel.block_boundaries:
            cut[p] = 1
        pin = np.zeros(n, dtype=np.uint8)
        if pinned is not None:
            for i in pinned:
                pin[i] = 1
        gids = np.array([i for i, ins in enumerate(sched) if ins.klass in GLOBAL_CLASSES],
                        dtype=np.int32)
        refs_np = np.frombuffer(refs, dtype=np.uint8).copy()
        return cls(n, words, ctrl, lat, klass, reads.reshape(-1), writes.reshape(-1),
                   refs_np, nrefs, cut, pin, gids, tuple(intern))
