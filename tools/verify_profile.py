"""Per-phase device time of one verifier batch (fill, baseline run, candidate run, compare)."""
import sys, time, ctypes
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2403_16863_b200.verify import Verifier
from paper_2403_16863_b200.engine import CmpResult

for kind in ("gemm", "attn"):
    v = Verifier(kind)
    ident = np.arange(v.module.n, dtype=np.uint16)
    v.run(ident, 2 * v.batch)
    ctx = v.ctx
    def t(fn, n=5):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(n): fn()
        torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
    res = CmpResult()
    nbytes = sum(x.numel() * 2 for x in v.target.inputs)
    tf = t(lambda: v.target.fill(stream=3))
    tr = t(lambda: v._run(None, v.launch_ref))
    tc = t(lambda: v._run(ident, v.launch_cand))
    tcmp = t(lambda: ctx.lib.sip_compare(ctx.handle, ctypes.c_void_p(v.out_ref.data_ptr()),
                                         ctypes.c_void_p(v.out_cand.data_ptr()), v.out_ref.numel(), 0,
                                         v.atol, v.rtol, v.elems_per_sample, 0, ctypes.byref(res)))
    tb = t(lambda: v.run(ident, v.batch), 3)
    print(f"{kind}: batch {v.batch}: fill {tf:.3f} ms ({nbytes/tf/1e6:.0f} GB/s), ref {tr:.3f}, cand {tc:.3f}, "
          f"compare {tcmp:.3f} ({4*v.out_ref.numel()/tcmp/1e6:.0f} GB/s), whole batch {tb:.3f} ms", flush=True)
