"""Where a hardware-search round's time goes (bench hw-phase shape: GEMM 4096^3, 16 chains)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2403_16863_b200 import AnnealConfig
from paper_2403_16863_b200.evaluator import B200Backend
from paper_2403_16863_b200.hwsearch import HardwareSearch
from paper_2403_16863_b200.targets import make_target
tgt = make_target("gemm").allocate()
be = B200Backend(tgt, warmup=2, flush_l2=True)
cfg = AnnealConfig(seed=0, t_max=0.02, t_min=0.0005, cooling=1.02, measure_reps=5, candidate_classes="extended")
hs = HardwareSearch(be, cfg, 16)
acc = {"propose": 0.0, "measure": 0.0, "resolve": 0.0}
n = 0
for r in range(24):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    lo, cand = hs.chains.propose(with_schedules=True)
    t1 = time.perf_counter()
    live = np.nonzero(lo >= 0)[0]
    if len(live):
        smp = be.measure_batch(cand[live], cfg.measure_reps)
        t2 = time.perf_counter()
        for c, s in zip(live, smp):
            hs.times[c] = s.value; hs.status[c] = 1
        hs.chains.resolve(hs.times, hs.status)
        torch.cuda.synchronize(); t3 = time.perf_counter()
        acc["propose"] += t1 - t0; acc["measure"] += t2 - t1; acc["resolve"] += t3 - t2; n += len(live)
print({k: round(v * 1e3 / 24, 3) for k, v in acc.items()}, "ms per round;", n, "candidates", flush=True)
