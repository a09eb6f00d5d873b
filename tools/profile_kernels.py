"""Launch each hot kernel a few times for ncu captures (never used for timing)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
which = sys.argv[1]
if which == "gemm":
    from paper_2403_16863_b200.targets import GemmTarget
    from paper_2403_16863_b200.evaluator import B200Backend
    be = B200Backend(GemmTarget(M=4096, N=4096, K=4096).allocate())
    for _ in range(3):
        be.run_perm(None)
elif which == "attn":
    from paper_2403_16863_b200.attention import AttnTarget
    from paper_2403_16863_b200.evaluator import B200Backend
    be = B200Backend(AttnTarget(B=4, H=32, S=4096, D=128).allocate())
    for _ in range(3):
        be.run_perm(None)
elif which == "engine":
    from bench import decoded_listing
    from paper_2403_16863_b200 import AnnealConfig
    from paper_2403_16863_b200.engine import get_context
    from paper_2403_16863_b200.machine import MachineConfig
    from paper_2403_16863_b200.tables import KernelTables
    L = decoded_listing()
    dk = get_context().kernel(KernelTables.build(L.kernel, MachineConfig()))
    temps = AnnealConfig().temperatures()
    C = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    C = C or 112 * 128 * get_context().sm_count  # the bench default (bench.py)
    for r in range(2):  # the bench's epoch call (history recorded); ncu captures the second
        res, _ = dk.anneal_epoch_reduced(r * C, C, temps)
        print("launch", r, "chains", C, "priced", res["priced"], "replayed", res["replayed"], flush=True)
elif which == "verify":
    from paper_2403_16863_b200.verify import Verifier
    v = Verifier("gemm")
    ident = np.arange(v.module.n, dtype=np.uint16)
    v.run(ident, 3 * v.batch)
torch.cuda.synchronize()
print("done", which)
