"""A/B/C of attention cubin variants in one process (same inputs, same launch)."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2403_16863_b200.attention import AttnTarget
from paper_2403_16863_b200.cubin import Module, schedule_perm
from paper_2403_16863_b200.engine import get_context
import ctypes, numpy as np
variants = {"current": "paper_2403_16863_b200/targets/attn_fwd.cubin"}
threads = {}
for a in sys.argv[1:]:
    path, _, nt = a.partition("@")  # path@384: launch with 384 threads (older 1-warp-per-row layout)
    variants[path.split("/")[-1]] = path
    if nt:
        threads[path.split("/")[-1]] = int(nt)
import os
tgt = AttnTarget(B=int(os.environ.get("AB_B", 4)), H=32, S=int(os.environ.get("AB_S", 4096))).allocate()
ctx = get_context()
mods = {k: Module(open(v, 'rb').read(), "attn_fwd_f16", ctx=ctx) for k, v in variants.items()}
import statistics
res = {k: [] for k in mods}
names = list(mods)
rounds = int(os.environ.get("AB_ROUNDS", 3))
for rnd in range(rounds):
    order = names[rnd % len(names):] + names[: rnd % len(names)]  # rotate: no variant always last
    for k in order:
        m = mods[k]
        lp, params = tgt.launch()
        if k in threads:  # the non-persistent layout: (S/256, B*H) grid of 384-thread CTAs
            lp.block[0] = threads[k]
            lp.grid[0], lp.grid[1] = tgt.S // 256, tgt.B * tgt.H
            lp.smem_bytes = 6 * 128 * 128 * 2 + 1024 + 144 + 4096
        if os.environ.get("AB_SMEM"):  # variants with deeper rings: give every variant this much
            lp.smem_bytes = int(os.environ["AB_SMEM"])
        med = ctypes.c_double(); raw = np.zeros(10)
        ctx.check(ctx.lib.sip_measure(m.handle, None, ctypes.byref(lp), 2, 10, 0, ctypes.byref(med),
                                      raw.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        res[k].append(tgt.flops / med.value / 1e9)
        if rounds <= 3:
            print(f"{k:20s} {med.value*1e3:8.1f} us  {tgt.flops/med.value/1e9:7.1f} TFLOP/s", flush=True)
for k in names:
    print(f"{k:20s} median over {rounds} rounds: {statistics.median(res[k]):7.1f} TFLOP/s "
          f"(min {min(res[k]):.0f}, max {max(res[k]):.0f})", flush=True)
