"""Engine time split: one launch with budget 1 (seeding + start checkpoints + one
iteration) vs the full 95-iteration budget, same chains."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
from bench import decoded_listing
from paper_2403_16863_b200 import AnnealConfig
from paper_2403_16863_b200.engine import get_context
from paper_2403_16863_b200.machine import MachineConfig
from paper_2403_16863_b200.tables import KernelTables

L = decoded_listing()
dk = get_context().kernel(KernelTables.build(L.kernel, MachineConfig()))
temps = AnnealConfig().temperatures()
C = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
for name, tt in (("budget 1", temps[:1]), ("budget 8", temps[:8]), ("budget 95", temps)):
    for _ in range(2):
        dk.anneal_epoch_reduced(0, C, tt)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for r in range(5):
        res, _ = dk.anneal_epoch_reduced(r * C, C, tt)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 5 * 1e3
    print(f"{name}: {ms:.2f} ms per launch, priced {res['priced']}, replayed {res['replayed']}", flush=True)
