"""Fused-kernel cost with and without per-iteration history records (262k chains)."""
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
C = 262144
def timed(fn, n=4):
    fn(0); torch.cuda.synchronize(); t0 = time.perf_counter()
    for r in range(n): fn(r + 1)
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
print("no history (epoch_reduced):", round(timed(lambda r: dk.anneal_epoch_reduced(r * C, C, temps)), 2), "ms", flush=True)
def keep(r):
    summ, res = dk.anneal_keep(np.arange(C, dtype=np.int64) + r * C, temps)
    del res
print("with history (anneal_keep):", round(timed(keep), 2), "ms", flush=True)
