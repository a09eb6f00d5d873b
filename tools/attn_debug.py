"""One small attention launch of a cubin variant (path[@threads]) vs torch; run under `timeout`."""
import sys, ctypes
sys.path.insert(0, '.')
import torch
from paper_2403_16863_b200.attention import AttnTarget
from paper_2403_16863_b200.cubin import Module
from paper_2403_16863_b200.engine import get_context

path, _, nt = sys.argv[1].partition("@")
S = int(sys.argv[2]) if len(sys.argv) > 2 else 512
tgt = AttnTarget(B=1, H=2, S=S).allocate()
ctx = get_context()
m = Module(open(path, "rb").read(), "attn_fwd_f16", ctx=ctx)
lp, params = tgt.launch()
if nt:
    lp.block[0] = int(nt)
ctx.check(ctx.lib.sip_run(m.handle, None, ctypes.byref(lp)))
torch.cuda.synchronize()
ref = tgt.reference_output()
print(path, "max abs err", (tgt.output.float() - ref).abs().max().item(), flush=True)
