"""Time GEMM cubin variants (same launch, same inputs) at 4096^3: path arguments."""
import ctypes, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2403_16863_b200.cubin import Module
from paper_2403_16863_b200.engine import get_context, c_dblp
from paper_2403_16863_b200.targets import GemmTarget

tgt = GemmTarget(M=4096, N=4096, K=4096).allocate()
ctx = get_context()
variants = {"current": "paper_2403_16863_b200/targets/gemm_lrelu.cubin"}
for a in sys.argv[1:]:
    variants[a.split("/")[-1]] = a
mods = {k: Module(open(v, 'rb').read(), "gemm_lrelu_f16", ctx=ctx) for k, v in variants.items()}
for rnd in range(3):
    for k, m in mods.items():
        lp, params = tgt.launch()
        med = ctypes.c_double(); raw = np.zeros(20)
        ctx.check(ctx.lib.sip_measure(m.handle, None, ctypes.byref(lp), 2, 20, 1, ctypes.byref(med),
                                      raw.ctypes.data_as(c_dblp)))
        print(f"{k:28s} {med.value*1e3:8.1f} us  {tgt.flops/med.value/1e9:7.1f} TFLOP/s", flush=True)
