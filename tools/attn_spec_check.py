"""Speculative first-half exponentials (-DSIP_SPEC_EXP): outputs bit-identical to the
shipped attention cubin on the same inputs (several shapes, including a sigma that makes
row maxima grow past the rescale threshold), then the timing A/B (tools/attn_ab.py)."""
import ctypes, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2403_16863_b200.attention import AttnTarget
from paper_2403_16863_b200.cubin import Module
from paper_2403_16863_b200.engine import get_context

ctx = get_context()
base = Module(open("paper_2403_16863_b200/targets/attn_fwd.cubin", "rb").read(), "attn_fwd_f16", ctx=ctx)
spec = Module(open(sys.argv[1], "rb").read(), "attn_fwd_f16", ctx=ctx)
for (B, H, S, sigma) in [(4, 32, 4096, 0.5), (2, 15, 4096, 0.5), (1, 4, 16384, 0.5), (1, 8, 1024, 3.0), (2, 4, 2048, 8.0)]:
    tgt = AttnTarget(B=B, H=H, S=S, sigma=sigma).allocate()
    outs = []
    for m in (base, spec):
        tgt.output.zero_()
        lp, params = tgt.launch()
        ctx.check(ctx.lib.sip_run(m.handle, None, ctypes.byref(lp)))
        torch.cuda.synchronize()
        outs.append(tgt.output.clone())
    same = torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))
    print(f"B{B} H{H} S{S} sigma {sigma}: bit-identical {same}", flush=True)
