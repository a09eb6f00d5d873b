"""Engine throughput vs chains per GPU (exploratory)."""
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
for C in [8192, 32768, 65536, 131072, 262144]:
    dk.anneal_epoch(np.arange(C), temps, with_history=False)
    torch.cuda.synchronize()
    t = time.perf_counter(); pr = 0
    for r in range(3):
        _, summ, _, _ = dk.anneal_epoch(np.arange(C) + (r + 1) * C, temps, with_history=False)
        pr += int(summ["priced"].sum())
    dt = time.perf_counter() - t
    print(f"C={C:7d}: {pr/dt/1e6:8.1f} M candidates/s  ({dt/3*1e3:.1f} ms/epoch)", flush=True)
