"""Hardware search with the extended classes; print the moved instructions of every
ranked schedule that fails a verification screen (legality-model holes)."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2403_16863_b200 import AnnealConfig
from paper_2403_16863_b200.evaluator import B200Backend
from paper_2403_16863_b200.hwsearch import HardwareSearch
from paper_2403_16863_b200.targets import make_target
from paper_2403_16863_b200.verify import Verifier

kind = sys.argv[1] if len(sys.argv) > 1 else "gemm"
shape = dict(M=4096, N=4096, K=4096) if kind == "gemm" else dict(B=4, H=32, S=4096)
tgt = make_target(kind, **shape).allocate()
be = B200Backend(tgt)
cfg = AnnealConfig(seed=0, t_max=0.02, t_min=0.0005, cooling=1.02, measure_reps=5, candidate_classes="extended")
hs = HardwareSearch(be, cfg, 16, epoch=0)
for r in range(40):
    hs.step()
ver = Verifier(kind, batch=64)
seq = be.kernel.schedule
txt = lambda i: (seq[i].source_text or '').split(';')[0].strip()
for e, seed, sched in hs.ranked()[:12]:
    vr = ver.run(sched, 256, fail_fast=True, check_every=1)
    moved = [p for p in range(len(sched)) if sched[p] != p]
    print(f"energy {e:.4f} ok={vr.ok} maxerr={vr.max_abs_err:.3g} moved={len(moved)}", flush=True)
    if not vr.ok:
        for p in moved:
            print(f"   pos {p:5d} <- {int(sched[p]):5d} {txt(int(sched[p]))}")
