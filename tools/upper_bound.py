"""Per-configuration bounds on what reordering the movable instructions can buy.

For each tuning configuration the shipped cubin is timed against ablation builds in
which the region holding the search's movable instructions is made free
(build.py CUBIN_VARIANTS): GEMM -- the epilogue's LeakyReLU/packing ALU work removed
(`nomath`), the whole epilogue removed (`noepi`); attention -- the softmax's row max and
exponentials removed (`nomath`).  No reordering of those instructions can make them cost
less than nothing, so T_nvcc / T_ablation bounds the speed-up a schedule search over them
can reach.  Builds alternate round by round (L2 flushed before every launch, medians).

    python tools/upper_bound.py gpurun_out/upper_bound.json
"""
import ctypes
import json
import statistics
import sys

sys.path.insert(0, '.')
import numpy as np

from paper_2403_16863_b200.cubin import Module
from paper_2403_16863_b200.engine import c_dblp, get_context
from paper_2403_16863_b200.targets import TARGET_DIR, make_target

CONFIGS = [
    ("gemm", dict(M=4096, N=4096, K=4096), "gemm_lrelu_f16", ["gemm_lrelu", "gemm_lrelu_nomath", "gemm_lrelu_noepi"]),
    ("gemm", dict(M=512, N=512, K=2048), "gemm_lrelu_f16", ["gemm_lrelu", "gemm_lrelu_nomath", "gemm_lrelu_noepi"]),
    ("attn", dict(B=4, H=32, S=4096, D=128), "attn_fwd_f16", ["attn_fwd", "attn_fwd_nomath"]),
    ("attn", dict(B=4, H=32, S=1024, D=128), "attn_fwd_f16", ["attn_fwd", "attn_fwd_nomath"]),
    ("attn", dict(B=1, H=4, S=16384, D=128), "attn_fwd_f16", ["attn_fwd", "attn_fwd_nomath"]),
]
ROUNDS, REPS = 7, 15

ctx = get_context()
rows = []
for kind, shape, func, builds in CONFIGS:
    tgt = make_target(kind, **shape).allocate()
    lp, params = tgt.launch()
    mods = {b: Module((TARGET_DIR / f"{b}.cubin").read_bytes(), func, ctx=ctx) for b in builds}
    times = {b: [] for b in builds}
    for r in range(ROUNDS):
        order = builds[r % len(builds):] + builds[: r % len(builds)]
        for b in order:
            med = ctypes.c_double()
            raw = np.zeros(REPS)
            ctx.check(ctx.lib.sip_measure(mods[b].handle, None, ctypes.byref(lp), 2, REPS, 1, ctypes.byref(med),
                                          raw.ctypes.data_as(c_dblp)))
            times[b].append(med.value)
    t = {b: statistics.median(v) for b, v in times.items()}
    base = builds[0]
    row = {"kind": kind, "shape": shape, "nvcc_ms": t[base], "tflops": tgt.flops / t[base] / 1e9,
           "ablations_ms": {b: t[b] for b in builds[1:]},
           "speedup_bound": {b: t[base] / t[b] for b in builds[1:]},
           "rounds_ms": {b: v for b, v in times.items()}}
    rows.append(row)
    print(json.dumps({k: row[k] for k in ("kind", "shape", "nvcc_ms", "speedup_bound")}), flush=True)
    del tgt, mods
doc = {"what": __doc__.strip().splitlines()[0], "rounds": ROUNDS, "reps": REPS, "rows": rows}
if len(sys.argv) > 1:
    json.dump(doc, open(sys.argv[1], "w"), indent=1)
