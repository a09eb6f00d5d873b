import sys
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
for b in (1, 95):
    for r in range(3):
        dk.anneal_epoch_reduced(r * 262144, 262144, temps[:b])
torch.cuda.synchronize()
