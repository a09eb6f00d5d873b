"""Small launches of every libsip kernel family, for compute-sanitizer (memcheck,
racecheck, synccheck).  Sizes are tiny: the sanitizer serialises and instruments."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2403_16863_b200 import AnnealConfig, SimulatorBackend, parse_kernel, run_search
from paper_2403_16863_b200.engine import get_context
from paper_2403_16863_b200.machine import MachineConfig
from paper_2403_16863_b200.tables import KernelTables

which = sys.argv[1] if len(sys.argv) > 1 else "engine"
if which == "engine":
    from bench import decoded_listing
    L = decoded_listing()
    t = KernelTables.build(L.kernel, MachineConfig())
    dk = get_context().kernel(t)
    temps = AnnealConfig().temperatures()
    dk.anneal_epoch(np.arange(64, dtype=np.int64), temps)           # fused + history
    dk.anneal_epoch_reduced(64, 64, temps)                          # device epoch reduction
    summ, res = dk.anneal_keep(np.arange(32, dtype=np.int64), temps)
    res.fetch(3)
    ch = dk.chains(list(range(8)), [1000.0] * 8, temps, False, True, 8)  # step mode
    for _ in range(3):
        lo, cand = ch.propose(with_schedules=True)
        ch.resolve(np.where(lo >= 0, 1000.0, 0.0), np.where(lo >= 0, 1, 3).astype(np.uint8))
    dk.legality(np.tile(np.arange(dk.n, dtype=np.uint16), (4, 1)), [1, 2, 3, 4], hw_safe=True, min_fixed=8)
    hide = parse_kernel("[B------:R-:W0:-:S01] LDG.E R4, [R2.64] ;\n[B0-----:R-:W-:-:S01] IADD3 R5, R4, 0x1, RZ ;\n"
                        "[B------:R-:W-:-:S08] IADD3 R20, RZ, 0x1, RZ ;\n")
    run_search(hide, SimulatorBackend(), AnnealConfig(seed=0), chains=4)
elif which == "verify":
    from paper_2403_16863_b200.verify import Verifier
    v = Verifier("gemm", batch=4, shape=dict(M=256, N=256, K=256))
    v.run(np.arange(v.module.n, dtype=np.uint16), 8)
elif which == "attn_multi":
    # persistent attention with several items per CTA: 16 items on 3 CTAs (5-6 each), so
    # K/V ring phases, Q reloads and o_free hand-offs carry across items
    import os
    os.environ["SIP_ATTN_MAX_CTAS"] = "3"
    from paper_2403_16863_b200.evaluator import B200Backend
    from paper_2403_16863_b200.targets import make_target
    be = B200Backend(make_target("attn", B=1, H=8, S=512).allocate(), paired=False)
    assert be.launch.grid[0] == 3
    be.run_perm(None)
elif which in ("gemm", "attn"):
    from paper_2403_16863_b200.evaluator import B200Backend
    from paper_2403_16863_b200.targets import make_target
    shape = dict(M=256, N=512, K=256) if which == "gemm" else dict(B=1, H=1, S=512)
    be = B200Backend(make_target(which, **shape).allocate(), paired=False)
    be.run_perm(None)
print("done", which)
