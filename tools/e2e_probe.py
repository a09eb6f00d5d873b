"""Host time per anneal_keep_reduced call (e2e overhead probe): C chains, SlotRow or dense."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from bench import decoded_listing
from paper_2403_16863_b200 import AnnealConfig
from paper_2403_16863_b200.engine import get_context
from paper_2403_16863_b200.machine import MachineConfig
from paper_2403_16863_b200.tables import KernelTables
L = decoded_listing()
dk = get_context().kernel(KernelTables.build(L.kernel, MachineConfig()))
temps = AnnealConfig().temperatures()
hold = int(sys.argv[1])  # results kept alive across calls (1: the bench's e2e shape)
for C in [int(x) for x in sys.argv[2:]]:
    keep = []
    for r in range(6):
        torch.cuda.synchronize()
        t = time.perf_counter()
        res, dr = dk.anneal_keep_reduced(np.arange(C) + r * C, temps)
        t1 = time.perf_counter()
        keep.append(dr)
        while len(keep) > hold:
            keep.pop(0)
        t2 = time.perf_counter()
        print(f"C={C} call {r}: keep_reduced {1e3*(t1-t):.2f} ms, release {1e3*(t2-t1):.2f} ms", flush=True)
