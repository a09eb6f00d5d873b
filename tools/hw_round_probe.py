"""Where a hardware-search round's time goes at the bench's hw-phase shape (GEMM 4096^3,
128 chains, extended classes): host time per phase and, with SIP_EVAL_TIMING=1, the
evaluator's own split (load+warm-up enqueue / timed enqueue / execute) on stderr."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2403_16863_b200 import AnnealConfig
from paper_2403_16863_b200.evaluator import B200Backend
from paper_2403_16863_b200.hwsearch import HardwareSearch
from paper_2403_16863_b200.targets import make_target

kind = sys.argv[1] if len(sys.argv) > 1 else "gemm"
chains = int(sys.argv[2]) if len(sys.argv) > 2 else 128
tgt = make_target(kind).allocate()
be = B200Backend(tgt, warmup=2, flush_l2=True)
cfg = AnnealConfig(seed=0, t_max=0.02, t_min=0.0005, cooling=1.02, measure_reps=5, candidate_classes="extended")
hs = HardwareSearch(be, cfg, chains)
hs.step()
be.kernel_ms.clear()
acc = {"propose": 0.0, "measure": 0.0, "resolve": 0.0}
n = 0
R = 24
torch.cuda.synchronize()
w0 = time.perf_counter()
for r in range(R):
    t0 = time.perf_counter()
    lo, cand = hs.chains.propose(with_schedules=True)
    t1 = time.perf_counter()
    live = np.nonzero(lo >= 0)[0]
    if len(live):
        smp = be.measure_batch(cand[live], cfg.measure_reps)
        t2 = time.perf_counter()
        for c, s in zip(live, smp):
            hs.times[c] = s.value; hs.status[c] = 1
        hs.chains.resolve(hs.times, hs.status)
        t3 = time.perf_counter()
        acc["propose"] += t1 - t0; acc["measure"] += t2 - t1; acc["resolve"] += t3 - t2; n += len(live)
torch.cuda.synchronize()
wall = time.perf_counter() - w0
kern = list(be.kernel_ms)
tk = sum(kern) / len(kern)
roof = 1e3 / ((be.warmup + cfg.measure_reps) * tk)
print({k: round(v * 1e3 / R, 3) for k, v in acc.items()}, "ms per round;", n, "candidates;",
      f"rate {n / wall:.1f}/s, T_kernel {tk:.4f} ms, roofline {roof:.1f}/s, frac {n / wall / roof:.3f}", flush=True)
