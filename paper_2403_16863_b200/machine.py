"""Machine model configuration and the scoreboard energy.

``MachineConfig`` keeps the reference's parameters and latency lookup
(reference ``machine.py:33-92``).  ``simulate`` prices schedules with the
single-warp in-order scoreboard of reference ``machine.py:116-161``, but the
replay itself runs on the GPU (``csrc/engine.cu: sim_replay``); the host only
packs the per-instruction latency/control table once per kernel.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Mapping

from .ir import BARRIER_SLOTS, GLOBAL_CLASSES, Instruction, InstrClass, Kernel

DEFAULT_CPI = {"FFMA": 4, "IMAD": 5, "POPC": 15}
DEFAULT_CLASS_CPI = {
    InstrClass.COMPUTE: 4,
    InstrClass.SHARED_LOAD: 30,
    InstrClass.SHARED_STORE: 30,
    InstrClass.BARRIER: 1,
    InstrClass.CONTROL_FLOW: 1,
    InstrClass.OTHER: 4,
}


@dataclass(frozen=True)
class MachineConfig:
    global_mem_latency: int = 400
    barrier_count: int = BARRIER_SLOTS
    issue_width: int = 1
    cpi_table: Mapping = field(default_factory=lambda: dict(DEFAULT_CPI))
    class_cpi: Mapping = field(default_factory=lambda: dict(DEFAULT_CLASS_CPI))
    shared_size: int = 64 * 1024

    def __post_init__(self) -> None:
        if self.issue_width != 1:
            raise ValueError("only issue_width 1 is modeled")
        if self.global_mem_latency < 1:
            raise ValueError("global_mem_latency must be >= 1")
        for key, cpi in self.cpi_table.items():
            if cpi < 1:
                raise ValueError(f"cpi for {key!r} must be >= 1")

    def latency_of(self, ins: Instruction) -> int:
        """Global classes -> memory latency; else longest-prefix CPI; else class CPI."""
        if ins.klass in GLOBAL_CLASSES:
            return self.global_mem_latency
        mnem = ins.mnemonic.upper()
        hits = [key for key in self.cpi_table if mnem.startswith(key)]
        if hits:
            return self.cpi_table[max(hits, key=len)]
        return self.class_cpi.get(ins.klass, 4)

    @classmethod
    def from_dict(cls, data: Mapping) -> "MachineConfig":
        kw = dict(data)
        if "cpi" in kw:
            kw["cpi_table"] = {str(k).upper(): int(v) for k, v in kw.pop("cpi").items()}
        if "class_cpi" in kw:
            kw["class_cpi"] = {InstrClass(k): int(v) for k, v in kw.pop("class_cpi").items()}
        return cls(**kw)


@dataclass(frozen=True)
class SimReport:
    total_cycles: int
    instruction_count: int
    stalls: tuple
    barrier_waits: Mapping

    def to_json(self) -> str:
        return json.dumps(
            {
                "total_cycles": self.total_cycles,
                "instruction_count": self.instruction_count,
                "stalls": [list(s) for s in self.stalls],
                "barrier_waits": {str(b): w for b, w in sorted(self.barrier_waits.items())},
            },
            sort_keys=True,
        )


def simulate(kernel: Kernel, config: MachineConfig | None = None) -> SimReport:
    """Scoreboard replay of one schedule on the GPU (see ``engine.simulate_schedules``)."""
    from .engine import KernelTables, get_context

    cfg = config or MachineConfig()
    if not kernel.schedule:
        return SimReport(0, 0, (), {})
    tables = KernelTables.build(kernel, cfg)
    dk = get_context().kernel(tables)
    totals, waited, binding = dk.simulate([tuple(range(len(kernel)))], detail=True)
    stalls = tuple((i, int(w)) for i, w in enumerate(waited[0]))
    bw: dict = {}
    for w, b in zip(waited[0], binding[0]):
        if w and b >= 0:
            bw[int(b)] = bw.get(int(b), 0) + int(w)
    return SimReport(int(totals[0]), len(kernel), stalls, bw)
