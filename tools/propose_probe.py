"""Time of one hardware-mode propose round (chains_propose_kernel) per candidate class."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2403_16863_b200 import AnnealConfig
from paper_2403_16863_b200.evaluator import B200Backend
from paper_2403_16863_b200.targets import make_target
be = B200Backend(make_target("gemm").allocate(), paired=False)
for classes in ["extended", "sm100"]:
    for C in [256, 4096]:
        t = be.tables_for(be.kernel, classes)
        dk = be.ctx.kernel(t)
        cfg = AnnealConfig(seed=0, t_max=0.01, t_min=0.01 / 40, cooling=1.02)
        temps = cfg.temperatures()
        ch = dk.chains(list(range(C)), [1.0] * C, temps, False, True, be.min_fixed)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lo, cand = ch.propose(with_schedules=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{classes:8s} C={C:5d}: propose {dt*1e3:8.2f} ms, live {int((lo >= 0).sum())}", flush=True)
