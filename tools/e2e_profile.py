import sys, time
sys.path.insert(0, '.')
import cProfile, pstats
from bench import decoded_listing
from paper_2403_16863_b200 import AnnealConfig, SimulatorBackend, run_search
from paper_2403_16863_b200.machine import MachineConfig
L = decoded_listing()
C = int(sys.argv[1]) if len(sys.argv) > 1 else 227328
for k in range(2):
    run_search(L.kernel, SimulatorBackend(MachineConfig()), AnnealConfig(seed=k * C), chains=C).best.state.best_perm
pr = cProfile.Profile(); pr.enable()
t0 = time.perf_counter()
for k in range(3):
    rep = run_search(L.kernel, SimulatorBackend(MachineConfig()), AnnealConfig(seed=(5 + k) * C), chains=C)
    rep.best.state.best_perm
print("per step ms", (time.perf_counter() - t0) / 3 * 1e3)
pr.disable(); pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
