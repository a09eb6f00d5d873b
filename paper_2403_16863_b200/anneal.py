"""Simulated annealing over SASS schedules (reference ``anneal.py``), on the GPU.

``anneal()`` keeps the reference signature and returns an ``AnnealState``
whose ``history_jsonl()`` is byte-identical to the reference for the same
seed and a deterministic backend.  Two execution paths, both on the device:

* simulator energy (``SimulatorBackend``, no tester): the complete chain --
  MT19937 draws, proposal, O(1) legality, scoreboard replay, Metropolis --
  runs in one kernel launch (``sip_anneal``);
* any other backend / a tester: *step mode* -- the device draws and vets
  proposals (``sip_chains_propose``), the host prices each legal candidate
  with ``backend.measure`` and feeds the time back (``sip_chains_resolve``).

The host only turns the compact per-iteration records into ``HistoryRecord``
objects (energy = t / t0, feedback = (t_prev - t) / t0, as ``anneal.py:191-193``).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass
from typing import Callable

import numpy as np

from .backends import MeasurementFailed, SimulatorBackend
from .engine import (ST_ACCEPTED, ST_MEASURE, ST_PRICED, ST_TEST, STATUS_REASON, get_context,
                     temperature_schedule)
from .ir import Kernel
from .machine import MachineConfig
from .perturb import NoCandidatesError, candidates
from .tables import KernelTables


class InvalidBaseline(Exception):
    """Baseline runtime must be strictly positive."""


def feedback(t0: float, t_prev: float, t_curr: float) -> float:
    """Eq. 1 of the paper: (t_prev - t_curr) / t0 (reference anneal.py:28-36)."""
    if t0 <= 0:
        raise InvalidBaseline(f"baseline {t0} is not positive")
    return (t_prev - t_curr) / t0


def accept_move(delta_e: float, temperature: float, rng) -> bool:
    """Metropolis rule (host utility; the device applies the same rule per chain)."""
    if delta_e < 0:
        return True
    return rng.random() < math.exp(-delta_e / temperature)


@dataclass(frozen=True)
class AnnealConfig:
    t_max: float = 1.0
    t_min: float = 0.01
    cooling: float = 1.05
    seed: int = 0
    measure_reps: int = 5
    tests_per_step: int = 0
    unsafe_moves: bool = False
    hw_safe: bool = False          # extension; False reproduces the reference
    min_fixed_distance: int = 8    # hw_safe: issue distance a fixed-latency RAW pair keeps
    candidate_classes: str = "global"  # "extended": sm_100 extension; global = reference

    def __post_init__(self) -> None:
        if self.t_min <= 0 or self.t_max <= 0:
            raise ValueError("temperatures must be positive")
        if self.t_min > self.t_max:
            raise ValueError("t_min must not exceed t_max")
        if self.cooling <= 1.0:
            raise ValueError("cooling factor must be > 1")
        if self.measure_reps < 3:
            raise ValueError("measure_reps must be >= 3")
        if self.tests_per_step < 0:
            raise ValueError("tests_per_step must be >= 0")

    @property
    def iteration_budget(self) -> int:
        if self.t_max == self.t_min:
            return 0
        return math.ceil(math.log(self.t_max / self.t_min) / math.log(self.cooling))

    def temperatures(self) -> np.ndarray:
        return temperature_schedule(self.t_max, self.cooling, self.iteration_budget)


@dataclass(frozen=True)
class HistoryRecord:
    iteration: int
    candidate: int
    direction: str
    energy: float | None
    feedback: float
    accepted: bool
    temperature: float
    rejected: str | None = None

    def to_json(self) -> str:
        return json.dumps({
            "iteration": self.iteration,
            "action": {"candidate": self.candidate, "direction": self.direction},
            "energy": self.energy,
            "feedback": self.feedback,
            "accepted": self.accepted,
            "temperature": self.temperature,
            "rejected": self.rejected,
        }, sort_keys=True)


def records_to_history(records, t0: float, temps) -> list:
    """Compact device records -> HistoryRecord list (energy/feedback as anneal.py:191-193)."""
    out = []
    t_prev = t0
    for it in range(len(records)):
        r = records[it]
        st = int(r["status"])
        direction = "down" if int(r["direction"]) else "up"
        if st in (ST_ACCEPTED, ST_PRICED):
            t = float(r["time"])
            acc = st == ST_ACCEPTED
            out.append(HistoryRecord(it, int(r["candidate"]), direction, t / t0,
                                     feedback(t0, t_prev, t), acc, float(temps[it])))
            if acc:
                t_prev = t
        else:
            out.append(HistoryRecord(it, int(r["candidate"]), direction, None, 0.0, False,
                                     float(temps[it]), rejected=STATUS_REASON[st]))
    return out


class AnnealState:
    """Search outcome; ``history`` is materialised lazily from device records."""

    def __init__(self, best: Kernel | None, best_energy: float, current: Kernel | None,
                 current_energy: float, baseline: float, unit: str, iterations: int, history=None,
                 *, records=None, temps=None, best_perm=None, current_perm=None, base=None,
                 ambiguous: int = 0, device=None, priced: int | None = None):
        self._best = best
        self._current = current
        self._base = base  # listing the permutations index into (kernels built on access)
        self._device = device  # (DeviceResults, chain): records/schedules still in HBM
        self._priced = priced
        self._current_perm = current_perm
        self.best_energy = best_energy
        self.current_energy = current_energy
        self.baseline = baseline
        self.unit = unit
        self.iterations = iterations
        self._history = history
        self._records = records
        self._temps = temps
        self._best_perm = best_perm
        self.ambiguous = ambiguous

    def _pull(self) -> None:
        if self._device is not None and self._records is None:
            res, c = self._device
            self._records, self._best_perm, self._current_perm = res.fetch(c)

    @property
    def best_perm(self):
        if self._best_perm is None:
            self._pull()
        return self._best_perm

    @property
    def current_perm(self):
        if self._current_perm is None:
            self._pull()
        return self._current_perm

    @property
    def best(self) -> Kernel:
        if self._best is None and self._base is not None and self.best_perm is not None:
            self._best = _permuted(self._base, self.best_perm)
        return self._best

    @property
    def current(self) -> Kernel:
        if self._current is None and self._base is not None and self.current_perm is not None:
            self._current = _permuted(self._base, self.current_perm)
        return self._current

    @property
    def history(self) -> list:
        if self._history is None:
            self._pull()
            self._history = ([] if self._records is None
                             else records_to_history(self._records, self.baseline, self._temps))
        return self._history

    @property
    def records(self):
        self._pull()
        return self._records

    @property
    def best_time(self) -> float:
        return self.best_energy * self.baseline

    @property
    def priced(self) -> int:
        if self._priced is not None:
            return self._priced
        if self.records is None:
            return sum(1 for r in self.history if r.energy is not None)
        return int(np.count_nonzero(self._records["status"] <= ST_PRICED))

    def history_jsonl(self) -> str:
        return "".join(rec.to_json() + "\n" for rec in self.history)


def _permuted(kernel: Kernel, perm) -> Kernel:
    seq = kernel.schedule
    return kernel.with_schedule(tuple(seq[int(i)] for i in perm))


_TABLES: dict = {}  # (id(kernel), machine, classes) -> (kernel, tables): listings are reused


_DEVICE_KERNELS: dict = {}


def device_kernel(kernel: Kernel, machine: MachineConfig | None = None, tables: KernelTables | None = None,
                  classes: str = "global"):
    if tables is None:
        key = (id(kernel), repr(machine or MachineConfig()), classes)
        hit = _TABLES.get(key)
        if hit is None or hit[0] is not kernel:
            if len(_TABLES) >= 8:
                _TABLES.pop(next(iter(_TABLES)))
            hit = (kernel, KernelTables.build(kernel, machine, classes=classes))
            _TABLES[key] = hit
        tables = hit[1]
    # one DeviceKernel per table set: its legality rows, baseline and chain workspace
    # (~10 KB per chain) are reused by later searches instead of rebuilt per call
    ctx = get_context()
    dkey = (id(tables), id(ctx))
    hit = _DEVICE_KERNELS.get(dkey)
    if hit is None or hit[0] is not tables:
        if len(_DEVICE_KERNELS) >= 4:
            _DEVICE_KERNELS.pop(next(iter(_DEVICE_KERNELS)))
        hit = (tables, ctx.kernel(tables))
        _DEVICE_KERNELS[dkey] = hit
    return hit[1]


class BatchStates:
    """The AnnealStates of one fused launch, built on access (a read-only list).

    Records, schedules and per-chain summaries stay in HBM until read: a state's
    energies come with its first access (one 48-byte summary), its history / best /
    current with theirs.  The champion and the priced total were reduced on the device.
    """

    def __init__(self, kernel: Kernel, reduced: dict, res, temps):
        self.kernel = kernel
        self.reduced = reduced
        self.res = res
        self.temps = temps
        self._summ = None
        self._states: dict = {}

    @property
    def summ(self) -> np.ndarray:
        """Every chain's summary (one device->host copy on first use)."""
        if self._summ is None:
            self._summ = self.res.summary()
        return self._summ

    def summary_of(self, c: int):
        return self._summ[c] if self._summ is not None else self.res.summary(c, 1)[0]

    @property
    def champion(self) -> int:
        """Chain index of the best (best energy, seed) -- driver.py:81-85's ranking."""
        return int(self.reduced["champion_chain"])

    def __len__(self) -> int:
        return self.res.C

    def __getitem__(self, c):
        if isinstance(c, slice):
            return [self[i] for i in range(*c.indices(len(self)))]
        if c < 0:
            c += len(self)
        if not 0 <= c < len(self):
            raise IndexError(c)
        st = self._states.get(c)
        if st is None:
            sm = self.summary_of(c)
            st = AnnealState(None, float(sm["best_energy"]), None, float(sm["current_energy"]),
                             float(sm["t0"]), "cycles", len(self.temps), temps=self.temps,
                             base=self.kernel, device=(self.res, c), priced=int(sm["priced"]),
                             ambiguous=int(sm["ambiguous"]))
            self._states[c] = st
        return st

    def __iter__(self):
        return (self[i] for i in range(len(self)))

    @property
    def priced_total(self) -> int:
        return int(self.reduced["priced"])


def anneal_batch_sim(kernel: Kernel, machine: MachineConfig, cfg: AnnealConfig, seeds,
                     tables: KernelTables | None = None, want_schedules: bool = True) -> list:
    """Many simulator-energy chains in one launch; one AnnealState per seed."""
    if len(candidates(kernel, cfg.candidate_classes)) == 0:
        raise NoCandidatesError("no global-memory instructions to move")
    dk = device_kernel(kernel, machine, tables, cfg.candidate_classes)
    temps = cfg.temperatures()
    reduced, res = dk.anneal_keep_reduced(seeds, temps, unsafe=cfg.unsafe_moves, hw_safe=cfg.hw_safe,
                                          min_fixed=cfg.min_fixed_distance)
    states = BatchStates(kernel, reduced, res, temps)
    if len(states):  # every chain's t0 is the listing's baseline (anneal.py:141-143)
        t0 = float(states[states.champion].baseline)
        if t0 <= 0:
            raise InvalidBaseline(f"baseline measurement {t0} is not positive")
    return states


def anneal_steps(kernel: Kernel, backend, cfg: AnnealConfig, seeds, *,
                 tester: Callable[[Kernel], bool] | None = None,
                 tables: KernelTables | None = None, on_epoch=None) -> list:
    """Step mode: device proposals, host pricing through ``backend.measure``.

    All chains advance together; each round prices at most one candidate per
    chain.  ``on_epoch(chains, round)`` may exchange schedules between rounds.
    """
    if len(candidates(kernel, cfg.candidate_classes)) == 0:
        raise NoCandidatesError("no global-memory instructions to move")
    seeds = list(seeds)
    t0 = []
    for _ in seeds:
        v = backend.measure(kernel, cfg.measure_reps).value
        if v <= 0:
            raise InvalidBaseline(f"baseline measurement {v} is not positive")
        t0.append(v)
    dk = device_kernel(kernel, MachineConfig(), tables, cfg.candidate_classes)
    temps = cfg.temperatures()
    chains = dk.chains(seeds, t0, temps, cfg.unsafe_moves, cfg.hw_safe, cfg.min_fixed_distance)
    C = len(seeds)
    times = np.zeros(C, dtype=np.float64)
    status = np.zeros(C, dtype=np.uint8)
    rnd = 0
    while True:
        lo, cand = chains.propose(with_schedules=True)
        live = np.nonzero(lo >= 0)[0]
        if len(live) == 0:
            break
        for c in live:
            cand_kernel = _permuted(kernel, cand[c])
            if tester is not None and not tester(cand_kernel):
                status[c], times[c] = ST_TEST, 0.0
                continue
            try:
                times[c] = backend.measure(cand_kernel, cfg.measure_reps).value
                status[c] = ST_PRICED
            except MeasurementFailed:
                status[c], times[c] = ST_MEASURE, 0.0
        chains.resolve(times, status)
        rnd += 1
        if on_epoch is not None:
            on_epoch(chains, rnd)
    hist, best, cur, summ = chains.result()
    unit = getattr(backend, "unit", "")
    return [AnnealState(None, float(summ["best_energy"][c]), None, float(summ["current_energy"][c]),
                        t0[c], unit, len(temps), records=hist[c], temps=temps, base=kernel,
                        best_perm=best[c], current_perm=cur[c], ambiguous=int(summ["ambiguous"][c]))
            for c in range(C)]


def uses_device_energy(backend) -> bool:
    """True when pricing is the stock scoreboard and may run entirely on the GPU."""
    return (getattr(backend, "device_energy", False)
            and type(backend).measure is SimulatorBackend.measure)


def anneal(kernel: Kernel, backend, config: AnnealConfig | None = None, *,
           tester: Callable[[Kernel], bool] | None = None) -> AnnealState:
    """One annealing chain (reference anneal.py:123-213), executed on the GPU."""
    cfg = config or AnnealConfig()
    if uses_device_energy(backend) and tester is None:
        return anneal_batch_sim(kernel, backend.machine, cfg, [cfg.seed])[0]
    from .driver import hardware_config

    cfg = hardware_config(backend, cfg)
    tables = backend.tables_for(kernel, cfg.candidate_classes) if hasattr(backend, "tables_for") else None
    return anneal_steps(kernel, backend, cfg, [cfg.seed], tester=tester, tables=tables)[0]
