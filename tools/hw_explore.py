"""Longer hardware-priced search on one target (exploration, prints a summary)."""
import argparse, sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2403_16863_b200 import AnnealConfig, candidates
from paper_2403_16863_b200.evaluator import B200Backend
from paper_2403_16863_b200.hwsearch import HardwareSearch
from paper_2403_16863_b200.targets import make_target
from paper_2403_16863_b200.verify import Verifier

ap = argparse.ArgumentParser()
ap.add_argument("--target", default="attn")
ap.add_argument("--classes", default="extended")
ap.add_argument("--chains", type=int, default=16)
ap.add_argument("--rounds", type=int, default=60)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--tmax", type=float, default=0.01)
a = ap.parse_args()
shape = dict(B=4, H=32, S=4096) if a.target == "attn" else dict(M=4096, N=4096, K=4096)
tgt = make_target(a.target, **shape).allocate()
be = B200Backend(tgt)
print("listing", be.listing.n, "candidates", len(candidates(be.kernel, a.classes)), flush=True)
cfg = AnnealConfig(seed=0, t_max=a.tmax, t_min=a.tmax / 40, cooling=1.02, measure_reps=a.reps,
                   candidate_classes=a.classes)
hs = HardwareSearch(be, cfg, a.chains, epoch=10)
t0 = time.time()
for r in range(a.rounds):
    hs.step()
    if r % 10 == 9:
        res = hs.result()
        print(f"round {r+1}: evaluated {hs.evaluated} best energy {res['best_energy']:.4f} "
              f"accepted {res['accepted']} ({time.time()-t0:.0f}s)", flush=True)
res = hs.result()
hist, *_ = hs.chains.result()
st = hist["status"]
print("status counts", {int(k): int((st == k).sum()) for k in np.unique(st)}, flush=True)
best = res["best_perm"]
ratio, raw = be.ratio(best, 45)
q1, q3 = np.percentile(raw, [25, 75])
print(f"re-timed speedup {1/ratio:.4f} (IQR {1/q3:.4f}-{1/q1:.4f}), moved {(best != be.identity).sum()}", flush=True)
vr = Verifier(a.target).run(best, 100_000)
print("verify", vr.to_dict(), flush=True)
