"""Oracle tables built from the reference's own per-instruction facts.

TEST INFRASTRUCTURE ONLY (like the rest of ``oracle/``): used by tests/ and by
bench.py's ``--impl reference`` / ``cpu_baseline`` legs, never by the product.

``tests/golden/targets.json.gz`` (``make_target_golden.py``) stores, for each
decoded target listing, what the *reference* computed per instruction:
``deps.reads_writes`` (``deps.py:68-199``), ``deps.mem_refs``
(``deps.py:215-249``), the class (``ir.classify``, ``ir.py:30-76``), the
scoreboard fields (``ir.ControlCode``, ``ir.py:84-118``), the latency
(``machine.MachineConfig.latency_of``, ``machine.py:76-85``) and the block
cuts (``sasstext.py:294-297``).  This module packs those facts into the
``sip_tables`` layout ``sip_oracle.c`` reads, so the reference arm runs the
oracle without touching the product's host frontend (``tables.py``).
"""
from __future__ import annotations

import gzip
import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
TARGETS = ROOT / "tests" / "golden" / "targets.json.gz"

MAX_REFS = 4
NO_BAR = 7
SPACE = {"global": 0, "shared": 1, "local": 2, "unknown": 3}
# reference ir.InstrClass values in declaration order (ir.py:18-27)
CLASSES = ["GlobalLoad", "GlobalStore", "GlobalAsyncCopy", "SharedLoad", "SharedStore",
           "Compute", "Barrier", "ControlFlow", "Other"]
GLOBAL = {"GlobalLoad", "GlobalStore", "GlobalAsyncCopy"}   # ir.GLOBAL_CLASSES (ir.py:30-32)
FENCE = {"Barrier", "ControlFlow"}                          # deps.py:336-343
MEMREF = np.dtype([("offset", "<i8"), ("base", "<i4"), ("size", "u1"), ("space", "u1"),
                   ("write", "u1"), ("pad", "u1")])


@dataclass
class GoldenTables:
    """Same field names as the product's KernelTables, which OracleListing reads."""
    n: int
    words: int
    ctrl: np.ndarray
    lat: np.ndarray
    klass: np.ndarray
    reads: np.ndarray
    writes: np.ndarray
    refs: np.ndarray
    nrefs: np.ndarray
    cut: np.ndarray
    pin: np.ndarray


def load_targets() -> dict:
    with gzip.open(TARGETS, "rt") as fh:
        return json.load(fh)["listings"]


def tables_from_facts(rec: dict) -> GoldenTables:
    n = rec["n"]
    intern: dict = {}

    def rid(name):
        return intern.setdefault(name, len(intern))

    for r, w in rec["rw"]:
        for name in sorted(set(r) | set(w)):
            rid(name)
    for lst in rec["refs"]:
        for space, base, off, size, write in lst:
            if base is not None:
                rid(base)
    words = max(1, (len(intern) + 63) // 64)
    reads = np.zeros((n, words), dtype=np.uint64)
    writes = np.zeros((n, words), dtype=np.uint64)
    for i, (r, w) in enumerate(rec["rw"]):
        for name in r:
            b = intern[name]
            reads[i, b >> 6] |= np.uint64(1 << (b & 63))
        for name in w:
            b = intern[name]
            writes[i, b >> 6] |= np.uint64(1 << (b & 63))
    refs = np.zeros(n * MAX_REFS, dtype=MEMREF)
    nrefs = np.zeros(n, dtype=np.uint8)
    for i, lst in enumerate(rec["refs"]):
        nrefs[i] = len(lst)
        for j, (space, base, off, size, write) in enumerate(lst):
            refs[i * MAX_REFS + j] = (int(off), -1 if base is None else intern[base], size, SPACE[space],
                                      int(write), 0)
    ctrl = np.zeros(n, dtype=np.uint32)
    for i, (c, klass) in enumerate(zip(rec["ctrl"], rec["classes"])):
        if c is None:
            wait, rd, wr, adv = 0, NO_BAR, NO_BAR, 1
        else:
            waits, rdb, wrb, stall = c
            wait = sum(1 << b for b in waits)
            rd = NO_BAR if rdb is None else rdb
            wr = NO_BAR if wrb is None else wrb
            adv = max(1, stall)  # machine.py:150: the issue pointer advances max(1, stall)
        glob = klass in GLOBAL
        ctrl[i] = (wait | (rd << 6) | (wr << 9) | (adv << 12) | (int(klass in FENCE) << 21)
                   | (int(glob) << 22) | (int(glob) << 23))
    cut = np.zeros(n + 1, dtype=np.uint8)
    for p in rec["cuts"]:
        cut[p] = 1
    return GoldenTables(n, words, ctrl, np.asarray(rec["lat"], dtype=np.uint32),
                        np.array([CLASSES.index(k) for k in rec["classes"]], dtype=np.uint8),
                        reads.reshape(-1), writes.reshape(-1), refs.view(np.uint8).copy(), nrefs, cut,
                        np.zeros(n, dtype=np.uint8))
