"""Hardware-priced search at scale on one target, recorded as JSON (profiles/).

Runs many annealing chains over the sm_100 extension classes until every chain has
spent its iteration budget (hwsearch.HardwareSearch, epoch exchange of the best),
then applies SIP's acceptance rule (the ranked schedules walked through a fail-fast
screen), re-times the accepted schedule against the nvcc one over 45 interleaved
pairs, and verifies it on 10 M samples.

    python tools/long_search.py --target gemm --chains 512 --out gpurun_out/long_gemm.json
"""
import argparse
import json
import sys
import time

sys.path.insert(0, '.')
import numpy as np

from paper_2403_16863_b200 import AnnealConfig, candidates
from paper_2403_16863_b200.evaluator import B200Backend
from paper_2403_16863_b200.hwsearch import HardwareSearch
from paper_2403_16863_b200.targets import make_target
from paper_2403_16863_b200.verify import Verifier

ap = argparse.ArgumentParser()
ap.add_argument("--target", default="gemm", choices=["gemm", "attn"])
ap.add_argument("--classes", default="extended")
ap.add_argument("--chains", type=int, default=512)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--tmax", type=float, default=0.01)
ap.add_argument("--epoch", type=int, default=10)
ap.add_argument("--max-seconds", type=float, default=900)
ap.add_argument("--verify-samples", type=int, default=10_000_000)
ap.add_argument("--cubin", default=None,
                help="attention cubin file in targets/ instead of the shipped one")
ap.add_argument("--shape", default=None, help="e.g. M=512,N=512,K=2048 or B=1,H=4,S=16384 (paper shapes)")
ap.add_argument("--out", required=True)
a = ap.parse_args()

shape = dict(B=4, H=32, S=4096) if a.target == "attn" else dict(M=4096, N=4096, K=4096)
if a.shape:
    shape.update({kv.split("=")[0]: int(kv.split("=")[1]) for kv in a.shape.split(",")})
extra = {"cubin_file": a.cubin} if a.cubin else {}
tgt = make_target(a.target, **shape, **extra).allocate()
be = B200Backend(tgt)
ncand = len(candidates(be.kernel, a.classes))
cfg = AnnealConfig(seed=0, t_max=a.tmax, t_min=a.tmax / 40, cooling=1.02, measure_reps=a.reps,
                   candidate_classes=a.classes)
hs = HardwareSearch(be, cfg, a.chains, epoch=a.epoch)
t0 = time.time()
rounds, trace = 0, []
while rounds < cfg.iteration_budget and time.time() - t0 < a.max_seconds:  # one iteration per chain per round
    hs.step()
    rounds += 1
    if rounds % 20 == 0:
        res = hs.result()
        trace.append({"round": rounds, "seconds": round(time.time() - t0, 1), "evaluated": hs.evaluated,
                      "best_energy": res["best_energy"]})
        print(trace[-1], flush=True)
search_s = time.time() - t0
res = hs.result()
ver = Verifier(a.target)
energy, best, rejected = hs.verified_best(ver)
ratio, raw = be.ratio(best, 45)
q1, q3 = np.percentile(raw, [25, 75])
vr = ver.run(best, a.verify_samples)
out = {
    "target": a.target, "shape": shape, "cubin": a.cubin or "shipped (-lineinfo)", "classes": a.classes, "candidates_in_listing": ncand,
    "listing_instructions": int(be.listing.n), "chains": a.chains, "rounds": rounds,
    "iteration_budget": cfg.iteration_budget, "evaluated": int(hs.evaluated),
    "search_seconds": round(search_s, 1), "candidates_per_s": hs.evaluated / search_s,
    "search_best_energy": float(res["best_energy"]), "accepted_energy": float(energy),
    "rejected_by_screen": [{"energy": float(e), "failed": int(v.failed)} for e, v in rejected],
    "retimed_speedup": 1.0 / ratio, "retimed_speedup_iqr": [1.0 / q3, 1.0 / q1], "pairs": 45,
    "instructions_moved": int((best != be.identity).sum()),
    "nvcc_ms": be.ref_ms, "nvcc_tflops": tgt.flops / be.ref_ms / 1e9, "cold_input_sets": be.nsets,
    "verify": {"samples": vr.samples, "passed": vr.passed, "failed": vr.failed,
               "bit_identical": vr.bitdiff_elems == 0, "seconds": round(vr.seconds, 2)},
    "trace": trace,
}
with open(a.out, "w") as fh:
    json.dump(out, fh, indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "trace"}), flush=True)
