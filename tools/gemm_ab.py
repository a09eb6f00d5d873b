"""A/B of the GEMM tail split in one process."""
import os, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2403_16863_b200.targets import GemmTarget
from paper_2403_16863_b200.evaluator import B200Backend
from paper_2403_16863_b200.cubin import schedule_perm
for split in ("1", "0", "1", "0"):
    os.environ["SIP_GEMM_SPLIT"] = split
    tgt = GemmTarget(M=4096, N=4096, K=4096).allocate()
    be = B200Backend(tgt, paired=False)
    s = be._measure_single(schedule_perm(be.kernel), 30)
    print(f"split={split}: {s.value*1e3:.1f} us {tgt.flops/s.value/1e9:.0f} TFLOP/s min {min(s.raw)*1e3:.1f}", flush=True)
