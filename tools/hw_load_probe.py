"""Does loading candidate modules cost device time?  One round of 64 GEMM candidates timed
cold (every module loaded in the call) and again with every module already cached; then
the hardware search with refill, its wall time split into propose / measure / resolve."""
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
hs = HardwareSearch(be, cfg, 64)
lo, cand = hs.chains.propose(with_schedules=True)
P = cand[lo >= 0][:64].copy()
k = len(P)
for label in ("cold", "cached", "cached"):
    be.kernel_ms.clear()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    be.measure_batch(P, 5)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    tk = sum(be.kernel_ms) / max(1, len(be.kernel_ms))
    dev = (k + 1) * 7 * tk
    print(f"{label}: k={k} wall {1e3*(t1-t0):.2f} ms, device work {dev:.2f} ms, busy {dev/(1e3*(t1-t0)):.3f}", flush=True)

hs = HardwareSearch(be, cfg, 128, refill=32)
hs.step()
import paper_2403_16863_b200.hwsearch as H
acc = {"propose": 0.0, "measure": 0.0, "resolve": 0.0}
orig_prop, orig_mb = hs._propose, be.measure_batch
def prop(co):
    t = time.perf_counter(); r = orig_prop(co); acc["propose"] += time.perf_counter() - t; return r
def mb(p, reps=5):
    t = time.perf_counter(); r = orig_mb(p, reps); acc["measure"] += time.perf_counter() - t; return r
hs._propose = prop
be.measure_batch = mb
be.kernel_ms.clear()
n0 = hs.evaluated
torch.cuda.synchronize(); w0 = time.perf_counter()
for _ in range(12):
    hs.step()
torch.cuda.synchronize(); wall = time.perf_counter() - w0
n = hs.evaluated - n0
tk = sum(be.kernel_ms) / len(be.kernel_ms)
print({k_: round(v * 1e3, 1) for k_, v in acc.items()}, f"wall {wall*1e3:.1f} ms, {n} priced, "
      f"{n / wall:.1f}/s, candidate device work {n * 7 * tk:.1f} ms, frac {n * 7 * tk / (wall * 1e3):.3f}", flush=True)
