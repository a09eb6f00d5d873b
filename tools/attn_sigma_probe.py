"""One cubin, one shape, large-magnitude inputs (rescale path taken often): does it finish,
and how far is it from fp32 torch?"""
import ctypes, sys
sys.path.insert(0, '.')
import torch
from paper_2403_16863_b200.attention import AttnTarget
from paper_2403_16863_b200.cubin import Module
from paper_2403_16863_b200.engine import get_context

path, B, H, S, sigma = sys.argv[1], *map(int, sys.argv[2:5]), float(sys.argv[5])
ctx = get_context()
m = Module(open(path, "rb").read(), "attn_fwd_f16", ctx=ctx)
tgt = AttnTarget(B=B, H=H, S=S, sigma=sigma).allocate()
lp, params = tgt.launch()
ctx.check(ctx.lib.sip_run(m.handle, None, ctypes.byref(lp)))
torch.cuda.synchronize()
ref = tgt.reference_output()
err = (tgt.output.float() - ref).abs().max().item()
print(path.split('/')[-1], B, H, S, sigma, "max abs err", err, "finite", bool(torch.isfinite(tgt.output).all()), flush=True)
