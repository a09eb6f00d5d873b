"""Per-candidate cost of the hardware-priced search as rounds accumulate loaded modules:
`python tools/eval_scaling.py attn 512` prints ms per priced candidate for three rounds of
512 chains (it should stay flat: DESIGN.md 6b)."""
import os
import sys
import time

sys.path.insert(0, '.')
from paper_2403_16863_b200 import AnnealConfig
from paper_2403_16863_b200.evaluator import B200Backend
from paper_2403_16863_b200.hwsearch import HardwareSearch
from paper_2403_16863_b200.targets import make_target

kind = sys.argv[1]
shape = dict(B=4, H=32, S=4096) if kind == "attn" else dict(M=4096, N=4096, K=4096)
be = B200Backend(make_target(kind, **shape).allocate())
cfg = AnnealConfig(seed=0, t_max=0.01, t_min=0.01 / 40, cooling=1.02, measure_reps=5, candidate_classes="extended")
for C in [int(x) for x in sys.argv[2:]]:
    hs = HardwareSearch(be, cfg, C, epoch=0)
    for r in range(int(os.environ.get("ROUNDS", 3))):
        t0 = time.perf_counter()
        n = hs.step()
        dt = time.perf_counter() - t0
        print(f"C={C} round {r}: priced {n} in {dt * 1e3:.0f} ms = {dt * 1e3 / max(n, 1):.2f} ms/candidate", flush=True)
