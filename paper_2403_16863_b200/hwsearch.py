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


class HardwareSearch:
    def __init__(self, backend, cfg: AnnealConfig, chains: int, *, seed0: int | None = None,
                 epoch: int = 0, dist=None):
        self.be = backend
        self.cfg = hardware_config(backend, cfg)
        self.kernel = backend.kernel
        self.tables = backend.tables_for(self.kernel, self.cfg.candidate_classes)
        self.dk = backend.ctx.kernel(self.tables)
        self.dist = dist  # a parallel.NcclGroup / TorchGroup when world_size > 1
        self.rank = dist.rank if dist else 0
        self.world = dist.world if dist else 1
        base = cfg.seed if seed0 is None else seed0
        self.seeds = [base + self.rank * chains + c for c in range(chains)]
        self.C = chains
        self.epoch = epoch
        self.rounds = 0
        self.evaluated = 0
        self.proposals_seen = 0
        ident = np.arange(self.dk.n, dtype=np.uint16)
        t0 = backend.measure_perm(ident, self.cfg.measure_reps).value
        self.t0 = t0
        self.temps = self.cfg.temperatures()
        self.chains = self.dk.chains(self.seeds, [t0] * chains, self.temps, self.cfg.unsafe_moves,
                                     self.cfg.hw_safe, self.cfg.min_fixed_distance)
        self.times = np.zeros(chains, dtype=np.float64)
        self.status = np.zeros(chains, dtype=np.uint8)
        self.launches = 0  # device kernels launched by this search (propose/resolve/evaluated runs)

    def step(self) -> int:
        """One round: propose, price every legal candidate, resolve.  Returns #priced."""
        lo, cand = self.chains.propose(with_schedules=True)
        self.launches += 1
        live = np.nonzero(lo >= 0)[0]
        n = 0
        if len(live) and hasattr(self.be, "measure_batch"):
            # every live chain's candidate timed in one CUDA graph (parallel cubin loads)
            samples = self.be.measure_batch(cand[live], self.cfg.measure_reps)
        else:
            samples = [self._measure(cand[c]) for c in live]
        for c, smp in zip(live, samples):
            if isinstance(smp, MeasurementFailed):
                self.times[c], self.status[c] = 0.0, ST_MEASURE
                continue
            self.times[c] = smp.value
            self.status[c] = ST_PRICED
            n += 1
            self.launches += (1 if getattr(self.be, "rounds", False) else 2) * (self.be.warmup + self.cfg.measure_reps)
        if n and getattr(self.be, "rounds", False):
            from .evaluator import ROUND_CHUNK
            chunks = -(-len(live) // ROUND_CHUNK)  # one nvcc reference per measured chunk
            self.launches += chunks * (self.be.warmup + self.cfg.measure_reps)
        if len(live):
            self.chains.resolve(self.times, self.status)
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

    def local_best(self):
        hist, best, cur, summ = self.chains.result()
        key = [(float(summ["best_energy"][c]), self.seeds[c]) for c in range(self.C)]
        c = min(range(self.C), key=lambda i: key[i])
        return key[c][0], key[c][1], best[c], hist, summ

    def exchange(self) -> None:
        """All-gather (energy, seed) per rank; every chain adopts the global best."""
        e, seed, sched, _, _ = self.local_best()
        if self.dist is None:
            self.chains.adopt(sched, e, e * self.t0)
            return
        be, _, _, sched = self.dist.exchange_best(e, seed, sched)
        self.chains.adopt(sched, be, be * self.t0)

    def ranked(self):
        """Distinct per-chain best schedules, best (energy, seed) first."""
        hist, best, cur, summ = self.chains.result()
        order = sorted(range(self.C), key=lambda c: (float(summ["best_energy"][c]), self.seeds[c]))
        seen, out = set(), []
        for c in order:
            key = best[c].tobytes()
            if key not in seen:
                seen.add(key)
                out.append((float(summ["best_energy"][c]), self.seeds[c], best[c]))
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
