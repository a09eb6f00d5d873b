"""Multi-chain search (reference ``driver.py:52-116``) with batched chains.

Chains ``seed .. seed+C-1`` are independent (``driver.py:73-79``).  The
reference runs them one after another; here

* simulator energy: all C chains run in ONE device launch (``sip_anneal``);
* hardware energy (``B200Backend``): all C chains advance together in step
  mode, the device proposing, the evaluator pricing one candidate per chain
  per round;
* any other backend (possibly stateful, e.g. a counting or failing test
  double): chains run sequentially in step mode, exactly in the reference's
  call order.

Ranking, verification and the store follow the reference unchanged:
champions are verified on the full plan, passing chains are ranked by
``(best_time, seed)``.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

from .anneal import AnnealConfig, AnnealState, anneal_batch_sim, anneal_steps, uses_device_energy
from .ir import Kernel
from .perturb import candidates
from .sasstext import serialize_kernel
from .store import ResultStore, input_hash


@dataclass
class ChainOutcome:
    seed: int
    state: AnnealState
    verdict: object | None

    @property
    def passed(self) -> bool:
        return True if self.verdict is None else self.verdict.ok


class LazyOutcomes:
    """ChainOutcomes of a batched simulator search, built on access (read-only list)."""

    def __init__(self, states, seed0: int):
        self.states = states
        self.seed0 = seed0
        self._items: dict = {}

    def __len__(self) -> int:
        return len(self.states)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        o = self._items.get(i)
        if o is None:
            o = self._items[i] = ChainOutcome(self.seed0 + i, self.states[i], None)
        return o

    def __iter__(self):
        return (self[i] for i in range(len(self)))


@dataclass
class SearchReport:
    kernel: Kernel
    input_digest: str
    baseline: float
    unit: str
    chains: list
    best: ChainOutcome | None
    candidate_count: int = 0

    @property
    def candidates_evaluated(self) -> int:
        """Priced proposals over all chains (history records with an energy)."""
        st = getattr(self.chains, "states", None)
        if st is not None and hasattr(st, "priced_total"):
            return st.priced_total
        return sum(o.state.priced for o in self.chains)

    @property
    def best_time(self) -> float | None:
        return None if self.best is None else self.best.state.best_time

    @property
    def improvement_pct(self) -> float | None:
        if self.best is None or self.baseline <= 0:
            return None
        return (self.baseline - self.best.state.best_time) / self.baseline * 100.0


def _tester(kernel, plan, cfg):
    if plan is None or cfg.tests_per_step <= 0:
        return None
    from .difftest import run_tests

    step_plan = replace(plan, samples=cfg.tests_per_step)
    return lambda cand: run_tests(kernel, cand, step_plan, fail_fast=True).ok


def hardware_config(backend, cfg: AnnealConfig) -> AnnealConfig:
    """Candidates that execute on the GPU must respect stall distances, reuse
    bits and pinned offsets; the extension is forced on.

    ``unsafe_moves`` (skip the dependency check, ``perturb.py:86-87``) is forced off:
    a RAW/WAR swap that runs as real SASS can write stray global memory or leave a
    sticky fault in the context the engine shares, and hw_safe only checks the
    neighbours of the swapped pair, not the pair itself."""
    if getattr(backend, "hardware", False):
        return replace(cfg, hw_safe=True, unsafe_moves=False,
                       min_fixed_distance=max(cfg.min_fixed_distance, backend.min_fixed))
    return cfg


def run_states(kernel: Kernel, backend, cfg: AnnealConfig, chains: int, tester=None,
               tables=None, on_epoch=None) -> list:
    cfg = hardware_config(backend, cfg)
    if tables is None and hasattr(backend, "tables_for"):
        tables = backend.tables_for(kernel, cfg.candidate_classes)
    if tester is None and uses_device_energy(backend):
        # consecutive seeds (driver.py:73-79) as a range: no per-chain host objects or arrays
        seeds = range(cfg.seed, cfg.seed + chains)
        return anneal_batch_sim(kernel, backend.machine, cfg, seeds, tables=tables)
    seeds = [cfg.seed + c for c in range(chains)]
    if getattr(backend, "batched_chains", False):
        return anneal_steps(kernel, backend, cfg, seeds, tester=tester, tables=tables,
                            on_epoch=on_epoch)
    states = []
    for s in seeds:
        states += anneal_steps(kernel, backend, replace(cfg, seed=s), [s], tester=tester,
                               tables=tables)
    return states


def run_search(kernel: Kernel, backend, anneal_cfg: AnnealConfig, *, chains: int = 1,
               plan=None, store: ResultStore | None = None, on_epoch=None) -> SearchReport:
    if chains < 1:
        raise ValueError("chains must be >= 1")
    digest = kernel.__dict__.get("_input_hash")  # frozen Kernel: hash its text once
    if digest is None:
        digest = kernel.__dict__["_input_hash"] = input_hash(serialize_kernel(kernel))
    states = run_states(kernel, backend, anneal_cfg, chains, _tester(kernel, plan, anneal_cfg),
                        on_epoch=on_epoch)
    if plan is None and store is None and hasattr(states, "champion"):
        # batched simulator search: the champion under (best_time, seed) (driver.py:81-85)
        # was reduced on the device -- every chain shares t0, so best_time orders like the
        # best energy; per-chain outcomes are built on access
        lazy = LazyOutcomes(states, anneal_cfg.seed)
        best = lazy[states.champion] if len(states) else None
        baseline = float(best.state.baseline) if best is not None else 0.0
        return SearchReport(kernel, digest, baseline, "cycles", lazy, best, len(candidates(kernel, anneal_cfg.candidate_classes)))
    outcomes = []
    for c, st in enumerate(states):
        verdict = None
        if plan is not None:
            from .difftest import run_tests

            verdict = run_tests(kernel, st.best, plan)
        outcomes.append(ChainOutcome(anneal_cfg.seed + c, st, verdict))
    baseline = states[-1].baseline if states else 0.0
    unit = states[-1].unit if states else getattr(backend, "unit", "")
    ranked = sorted((o for o in outcomes if o.passed), key=lambda o: (o.state.best_time, o.seed))
    best = ranked[0] if ranked else None

    if store is not None:
        entries = []
        for o in outcomes:
            vd = o.verdict.to_dict() if o.verdict is not None else {"skipped": True}
            store.write_chain(digest, o.seed, serialize_kernel(o.state.best), o.state.history_jsonl(), vd)
            entries.append({"seed": o.seed, "time": o.state.best_time, "passed": o.passed,
                            "iterations": o.state.iterations})
        store.update_manifest(digest, baseline=baseline, unit=unit, entries=entries)

    return SearchReport(kernel, digest, baseline, unit, outcomes, best, len(candidates(kernel, anneal_cfg.candidate_classes)))
