"""Hardware-search chain refill (``HardwareSearch(refill=R)``) on a B200.

* With deterministic pricing (the scoreboard simulator standing in for the timer), every
  chain of every refill cohort has exactly the history it has when its cohort runs on its
  own -- refill only adds independent chains (driver.py:73-79), it never changes one.
* With real hardware pricing, cohorts start as chains finish, seeds never repeat, and the
  search's priced count equals the priced records of all histories.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2403_16863_b200 import AnnealConfig  # noqa: E402
from paper_2403_16863_b200.backends import CostSample  # noqa: E402
from paper_2403_16863_b200.engine import ST_ACCEPTED, ST_PRICED  # noqa: E402
from paper_2403_16863_b200.evaluator import B200Backend  # noqa: E402
from paper_2403_16863_b200.hwsearch import HardwareSearch  # noqa: E402
from paper_2403_16863_b200.targets import GemmTarget  # noqa: E402

CFG = AnnealConfig(seed=5, t_max=0.02, t_min=0.0005, cooling=1.05, measure_reps=3,
                   candidate_classes="extended")


class SimPriced:
    """A B200Backend whose candidates are priced by the device scoreboard simulator
    (deterministic), so that two searches can be compared record for record."""

    def __init__(self, be):
        self._be = be
        self._dk = be.ctx.kernel(be.tables_for(be.kernel, CFG.candidate_classes))

    def __getattr__(self, name):
        return getattr(self._be, name)

    def _price(self, perms):
        return self._dk.simulate(np.asarray(perms, dtype=np.uint16))

    def measure_perm(self, perm, reps=5):
        return CostSample(float(self._price([perm])[0]), "cycles", reps, ())

    def measure_batch(self, perms, reps=5):
        return [CostSample(float(t), "cycles", reps, ()) for t in self._price(perms)]


@pytest.fixture(scope="module")
def backend():
    return B200Backend(GemmTarget(M=512, N=512, K=512).allocate())


def _run_to_end(hs, limit=400):
    for _ in range(limit):
        hs.step()
        if all(co.done for co in hs.cohorts):
            return
    raise AssertionError("search did not finish")


def test_refill_cohorts_equal_standalone_chains(backend):
    sp = SimPriced(backend)
    hs = HardwareSearch(sp, CFG, 16, refill=8)
    for _ in range(60):
        hs.step()
    finished = [co for co in hs.cohorts if co.done]
    assert len(hs.cohorts) > 2 and len(finished) >= 2
    for co in finished[:3]:
        alone = HardwareSearch(sp, CFG, len(co.seeds), seed0=co.seeds[0])
        assert alone.seeds == co.seeds
        _run_to_end(alone)
        h1, b1, _, s1 = hs._result_of(co)  # a finished cohort: fetched once, device chains released
        assert co.sc is None and co.final is not None
        h2, b2, _, s2 = alone.chains.result()
        assert np.array_equal(h1, h2)
        assert np.array_equal(b1, b2)
        assert np.array_equal(s1["best_energy"], s2["best_energy"])


def test_refill_keeps_rounds_full_on_hardware(backend):
    hs = HardwareSearch(backend, CFG, 16, refill=8)
    priced = [hs.step() for _ in range(30)]
    seeds = hs.seeds
    assert len(seeds) == len(set(seeds)) == 8 * len(hs.cohorts) and len(hs.cohorts) > 2
    hist, _, _, _ = hs._results()
    n_priced = int(np.count_nonzero((hist["status"] == ST_ACCEPTED) | (hist["status"] == ST_PRICED)))
    assert hs.evaluated == sum(priced) == n_priced
    # with refill, at least C - R chain slots are live in every round
    assert min(priced) >= 16 - 8
    e, seed, sched, _, _ = hs.local_best()
    assert seed in seeds and e <= 1.0 + 0.05
