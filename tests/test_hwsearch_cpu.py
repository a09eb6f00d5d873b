"""HardwareSearch bookkeeping on the CPU: cohorts, refill, seeds, result merging and the
release of finished cohorts, with a numpy stand-in for the device's step-mode chains
(the device chains themselves are covered by tests/test_hwsearch_gpu.py)."""
import numpy as np
import pytest

from paper_2403_16863_b200 import AnnealConfig
from paper_2403_16863_b200.backends import CostSample
from paper_2403_16863_b200.engine import RECORD_DTYPE, ST_ACCEPTED, ST_DEPENDENCY, ST_PRICED, SUMMARY_DTYPE
from paper_2403_16863_b200.hwsearch import HardwareSearch

N = 12  # instructions of the stand-in listing


class FakeChains:
    """Step-mode chains: a proposal is legal with probability 0.3 (an illegal one is
    recorded and spends an iteration, as on the device); accepted if not slower."""

    live = 0  # chain objects alive (device state held)

    def __init__(self, seeds, t0, temps):
        self.seeds = list(seeds)
        self.C, self.B = len(self.seeds), len(temps)
        self.rng = [np.random.default_rng(s) for s in self.seeds]
        self.it = np.zeros(self.C, dtype=np.int64)
        self.cur = np.tile(np.arange(N, dtype=np.uint16), (self.C, 1))
        self.best = self.cur.copy()
        self.e_x = np.ones(self.C)
        self.e_best = np.ones(self.C)
        self.t0 = t0[0]
        self.hist = np.zeros((self.C, self.B), dtype=RECORD_DTYPE)
        self.hist["status"] = 255
        self.lo = np.full(self.C, -1, dtype=np.int32)
        self.cand = np.zeros((self.C, N), dtype=np.uint16)
        FakeChains.live += 1

    def propose(self, with_schedules=True):
        for c in range(self.C):
            self.lo[c] = -1
            while self.it[c] < self.B:
                r = self.rng[c]
                lo = int(r.integers(0, N - 1))
                if r.random() < 0.3:
                    self.lo[c] = lo
                    row = self.cur[c].copy()
                    row[lo], row[lo + 1] = row[lo + 1], row[lo]
                    self.cand[c] = row
                    break
                self.hist[c, self.it[c]]["status"] = ST_DEPENDENCY
                self.it[c] += 1
        return self.lo, self.cand

    def resolve(self, times, status):
        for c in range(self.C):
            if self.lo[c] < 0:
                continue
            e = times[c] / self.t0
            acc = e <= self.e_x[c]
            if acc:
                self.cur[c] = self.cand[c]
                self.e_x[c] = e
                if e < self.e_best[c]:
                    self.e_best[c], self.best[c] = e, self.cand[c]
            self.hist[c, self.it[c]]["status"] = ST_ACCEPTED if acc else ST_PRICED
            self.hist[c, self.it[c]]["time"] = times[c]
            self.it[c] += 1
            self.lo[c] = -1

    def adopt(self, sched, energy, time):
        self.cur[:] = sched
        self.e_x[:] = energy

    def result(self):
        summ = np.zeros(self.C, dtype=SUMMARY_DTYPE)
        summ["best_energy"] = self.e_best
        return self.hist.copy(), self.best.copy(), self.cur.copy(), summ

    def __del__(self):
        FakeChains.live -= 1


class FakeKernel:
    n = N

    def chains(self, seeds, t0, temps, unsafe, hw_safe, min_fixed):
        return FakeChains(seeds, t0, temps)


class FakeCtx:
    def kernel(self, tables):
        return FakeKernel()


class FakeBackend:
    """Times a schedule by a fixed per-position cost (deterministic)."""

    hardware = False
    warmup = 2
    rounds = True
    kernel = None

    def __init__(self):
        self.ctx = FakeCtx()
        self.w = np.linspace(1.0, 2.0, N)
        self.batches = []

    def tables_for(self, kernel, classes="global"):
        return None

    def _t(self, perm):
        return float(np.dot(self.w, np.asarray(perm, dtype=np.float64)))

    def measure_perm(self, perm, reps=5):
        return CostSample(self._t(perm), "ms", reps, ())

    def measure_batch(self, perms, reps=5):
        self.batches.append(len(perms))
        return [CostSample(self._t(p), "ms", reps, ()) for p in perms]


CFG = AnnealConfig(seed=100, t_max=0.02, t_min=0.0005, cooling=1.2, measure_reps=3)


def test_single_cohort_keeps_reference_seeds():
    hs = HardwareSearch(FakeBackend(), CFG, 8)
    assert hs.seeds == list(range(100, 108)) and len(hs.cohorts) == 1
    while not hs.cohorts[0].done:
        hs.step()
    assert hs.chains is hs.cohorts[0].sc  # without refill nothing is released


def test_refill_spawns_cohorts_with_disjoint_seeds_and_full_rounds():
    be = FakeBackend()
    hs = HardwareSearch(be, CFG, 16, refill=4)
    priced = [hs.step() for _ in range(40)]
    seeds = hs.seeds
    assert len(seeds) == len(set(seeds)) == 4 * len(hs.cohorts) > 16
    assert min(priced[1:]) > 16 - 4  # at most R - 1 slots idle after a round's refill
    hist, best, cur, summ = hs._results()
    assert hist.shape[0] == len(seeds)
    n_priced = int(np.count_nonzero((hist["status"] == ST_ACCEPTED) | (hist["status"] == ST_PRICED)))
    assert hs.evaluated == sum(priced) == n_priced == sum(be.batches)


def test_refill_seeds_are_disjoint_across_ranks():
    class Rank:
        def __init__(self, r):
            self.rank, self.world = r, 2

    a = HardwareSearch(FakeBackend(), CFG, 8, refill=4, dist=Rank(0))
    b = HardwareSearch(FakeBackend(), CFG, 8, refill=4, dist=Rank(1))
    for _ in range(30):
        a.step()
        b.step()
    assert not set(a.seeds) & set(b.seeds)


def test_finished_cohorts_release_their_chains_and_keep_results():
    hs = HardwareSearch(FakeBackend(), CFG, 8, refill=4)
    for _ in range(40):
        hs.step()
    before = FakeChains.live
    e, seed, sched, hist, summ = hs.local_best()
    done = [co for co in hs.cohorts if co.done]
    assert done and all(co.sc is None and co.final is not None for co in done)
    assert FakeChains.live == before - len(done)
    # results of released cohorts are unchanged and still ranked
    e2, seed2, _, _, _ = hs.local_best()
    assert (e, seed) == (e2, seed2)
    ranked = hs.ranked()
    assert ranked[0][0] == e and ranked[0][1] == seed
    # exchange adopts into live cohorts only
    hs.exchange()
    for _ in range(5):
        hs.step()


def test_refill_must_divide_chains():
    with pytest.raises(ValueError):
        HardwareSearch(FakeBackend(), CFG, 10, refill=4)
