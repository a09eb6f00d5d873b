"""Hardware-energy search: many annealing chains per GPU, priced on the B200.

One process per GPU.  Each rank owns ``chains`` step-mode chains on its
device (``sip_chains_*``): every round the device proposes one legal move per
live chain (hw_safe legality), the evaluator times each candidate
(``sip_measure``), and the device applies the Metropolis rule.  Every
``epoch`` rounds the ranks all-gather their best (energy, seed) records over
NCCL and every chain adopts the global best schedule (the owner broadcasts
it) -- the north star's "allgather of (cost, schedule-id) each epoch".  With
one rank and exchange disabled this is exactly ``driver.run_search`` with a
``B200Backend``, chain for chain.

Reference anchors: chains with consecutive seeds (driver.py:73-79); ranking by
(best_time, seed) (driver.py:81-85); Metropolis/feedback (anneal.py:28-44).
"""
from __future__ import annotations

from dataclasses import replace

import numpy as np

from .anneal import AnnealConfig
from .driver import hardware_config
from .engine import ST_ACCEPTED, ST_MEASURE, ST_PRICED
from .backends import MeasurementFailed


class _Cohort:
    """A batch of step-mode chains created together (one ``sip_chains`` object)."""

    def __init__(self, sc, seeds):
        self.sc = sc
        self.seeds = list(seeds)
        self.C = len(self.seeds)
        self.times = np.zeros(self.C, dtype=np.float64)
        self.status = np.zeros(self.C, dtype=np.uint8)
        self.done = False  # every chain has spent its iteration budget
        self.final = None  # (hist, best, cur, summ) of a finished cohort, fetched once


class HardwareSearch:
    """``chains`` live chain slots per rank, priced together every round.

    ``refill=0`` (default): exactly ``chains`` chains with seeds ``base + rank*chains + c``
    -- ``driver.run_search`` with a ``B200Backend``, chain for chain.  ``refill=R``: the
    slots are kept busy at scale.  Chains finish at different rounds (an illegal proposal
    still spends an iteration, ``anneal.py:157-170``), so whenever at least R slots are
    idle a new cohort of R fresh seeds starts.  Every chain is still an independent
    reference chain of its own seed (``driver.py:73-79``); only more of them run, and every
    round prices a full set of candidates instead of the stragglers of one cohort.
    """

    def __init__(self, backend, cfg: AnnealConfig, chains: int, *, seed0: int | None = None,
                 epoch: int = 0, dist=None, refill: int = 0):
        self.be = backend
        self.cfg = hardware_config(backend, cfg)
        self.kernel = backend.kernel
        self.tables = backend.tables_for(self.kernel, self.cfg.candidate_classes)
        self.dk = backend.ctx.kernel(self.tables)
        self.dist = dist  # a parallel.NcclGroup / TorchGroup when world_size > 1
        self.rank = dist.rank if dist else 0
        self.world = dist.world if dist else 1
        self.base = cfg.seed if seed0 is None else seed0
        if refill and chains % refill:
            raise ValueError("chains must be a multiple of refill")
        self.refill = refill
        self.C = chains
        self.epoch = epoch
        self.rounds = 0
        self.evaluated = 0
        self.proposals_seen = 0
        ident = np.arange(self.dk.n, dtype=np.uint16)
        t0 = backend.measure_perm(ident, self.cfg.measure_reps).value
        self.t0 = t0
        self.temps = self.cfg.temperatures()
        self.cohorts = []
        self.launches = 0  # device kernels launched by this search (propose/resolve/evaluated runs)
        if refill:
            for _ in range(chains // refill):
                self._spawn()
        else:
            self._add([self.base + self.rank * chains + c for c in range(chains)])

    def _add(self, seeds):
        sc = self.dk.chains(seeds, [self.t0] * len(seeds), self.temps, self.cfg.unsafe_moves,
                            self.cfg.hw_safe, self.cfg.min_fixed_distance)
        co = _Cohort(sc, seeds)
        self.cohorts.append(co)
        return co

    def _spawn(self):
        g = len(self.cohorts)  # cohort g of rank r: seeds base + (g*world + r)*R + c, disjoint
        first = self.base + (g * self.world + self.rank) * self.refill
        return self._add(range(first, first + self.refill))

    @property
    def chains(self):
        """The first cohort's step-mode chains (the only one without refill)."""
        return self.cohorts[0].sc

    @property
    def seeds(self):
        return [s for co in self.cohorts for s in co.seeds]

    def _propose(self, co):
        lo, cand = co.sc.propose(with_schedules=True)
        self.launches += 1
        live = np.nonzero(lo >= 0)[0]
        if not len(live):
            co.done = True
        return live, cand

    def step(self) -> int:
        """One round: propose, price every legal candidate, resolve.  Returns #priced."""
        props = []
        for co in self.cohorts:
            if not co.done:
                live, cand = self._propose(co)
                if len(live):
                    props.append((co, live, cand))
        if self.refill:
            idle = self.C - sum(len(live) for _, live, _ in props)
            while idle >= self.refill:
                co = self._spawn()
                live, cand = self._propose(co)
                if len(live):
                    props.append((co, live, cand))
                idle -= len(live)
        n = 0
        if props:
            allc = np.concatenate([cand[live] for _, live, cand in props]) if len(props) > 1 \
                else props[0][2][props[0][1]]
            if hasattr(self.be, "measure_batch"):
                # every live chain's candidate timed in one round (parallel cubin loads)
                samples = self.be.measure_batch(allc, self.cfg.measure_reps)
            else:
                samples = [self._measure(p) for p in allc]
            i = 0
            for co, live, _ in props:
                for c in live:
                    smp = samples[i]
                    i += 1
                    if isinstance(smp, MeasurementFailed):
                        co.times[c], co.status[c] = 0.0, ST_MEASURE
                        continue
                    co.times[c] = smp.value
                    co.status[c] = ST_PRICED
                    n += 1
            self.launches += n * (1 if getattr(self.be, "rounds", False) else 2) * (self.be.warmup + self.cfg.measure_reps)
            if n and getattr(self.be, "rounds", False):
                from .evaluator import ROUND_CHUNK
                chunks = -(-len(allc) // ROUND_CHUNK)  # one nvcc reference per measured chunk
                self.launches += chunks * (self.be.warmup + self.cfg.measure_reps)
            for co, _, _ in props:
                co.sc.resolve(co.times, co.status)
                self.launches += 1
        self.rounds += 1
        self.evaluated += n
        if self.epoch and self.rounds % self.epoch == 0:
            self.exchange()
        return n

    def _measure(self, perm):
        try:
            return self.be.measure_perm(perm, self.cfg.measure_reps)
        except MeasurementFailed as exc:
            return exc

    def _result_of(self, co):
        if co.final is not None:
            return co.final
        res = co.sc.result()
        if co.done and self.refill:
            # a finished cohort never changes again (exchange adopts into live cohorts
            # only): keep its results on the host and release its device chains, so a long
            # refilled search holds device state for its live chains only
            co.final, co.sc = res, None
        return res

    def _results(self):
        """(hist, best, cur, summ) over every chain of every cohort, in seed-list order."""
        parts = [self._result_of(co) for co in self.cohorts]
        if len(parts) == 1:
            return parts[0]
        return tuple(np.concatenate([p[i] for p in parts]) for i in range(4))

    def local_best(self):
        hist, best, cur, summ = self._results()
        seeds = self.seeds
        key = [(float(summ["best_energy"][c]), seeds[c]) for c in range(len(seeds))]
        c = min(range(len(seeds)), key=lambda i: key[i])
        return key[c][0], key[c][1], best[c], hist, summ

    def exchange(self) -> None:
        """All-gather (energy, seed) per rank; every live chain adopts the global best."""
        e, seed, sched, _, _ = self.local_best()
        if self.dist is not None:
            e, _, _, sched = self.dist.exchange_best(e, seed, sched)
        for co in self.cohorts:
            if not co.done:
                co.sc.adopt(sched, e, e * self.t0)

    def ranked(self):
        """Distinct per-chain best schedules, best (energy, seed) first."""
        hist, best, cur, summ = self._results()
        seeds = self.seeds
        order = sorted(range(len(seeds)), key=lambda c: (float(summ["best_energy"][c]), seeds[c]))
        seen, out = set(), []
        for c in order:
            key = best[c].tobytes()
            if key not in seen:
                seen.add(key)
                out.append((float(summ["best_energy"][c]), seeds[c], best[c]))
        return out

    def verified_best(self, verifier, screen: int = 100_000, limit: int = 8):
        """SIP's acceptance rule (difftest.run_tests fail_fast): walk the
        ranked schedules and keep the first that passes a fail-fast screen of `screen`
        samples; schedules that fail are rejected.  Falls back to the nvcc schedule.
        Returns (energy, schedule, rejected list of (energy, VerifyResult))."""
        rejected = []
        ident = np.arange(self.dk.n, dtype=np.uint16)
        for e, _, sched in self.ranked()[:limit]:
            if e >= 1.0 or np.array_equal(sched, ident):
                break
            vr = verifier.run(sched, screen, fail_fast=True, check_every=8)
            if vr.ok:
                return e, sched, rejected
            rejected.append((e, vr))
        return 1.0, ident, rejected

    def result(self):
        e, seed, sched, hist, summ = self.local_best()
        priced = int(np.count_nonzero(hist["status"] <= ST_PRICED))
        accepted = int(np.count_nonzero(hist["status"] == ST_ACCEPTED))
        return {"best_energy": e, "best_seed": seed, "best_perm": sched, "priced": priced,
                "accepted": accepted, "t0_ms": self.t0, "summary": summ}
