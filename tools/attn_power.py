"""Clock and power while our attention kernel and torch SDPA each run back to back for ~3 s
(sustained, power-capped): TFLOP/s from the wall clock over 3 000 launches, SM clock and
board power medians from NVML every 20 ms."""
import sys, time, threading, ctypes
sys.path.insert(0, '.')
import numpy as np, torch
import pynvml
from paper_2403_16863_b200.attention import AttnTarget
from paper_2403_16863_b200.cubin import Module
from paper_2403_16863_b200.engine import get_context
import torch.nn.functional as F

pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
def sample(stop, out):
    while not stop.is_set():
        out.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(h) / 1000))
        time.sleep(0.02)
tgt = AttnTarget(B=4, H=32, S=4096).allocate()
ctx = get_context()
m = Module(tgt.cubin()[0], "attn_fwd_f16", ctx=ctx)
lp, params = tgt.launch()
q, k, v = tgt.inputs
def ours(n):
    for _ in range(n): ctx.check(ctx.lib.sip_run_async(m.handle, None, ctypes.byref(lp)))
def sdpa(n):
    for _ in range(n): F.scaled_dot_product_attention(q, k, v)
for name, fn in (("ours", ours), ("sdpa", sdpa), ("ours", ours), ("sdpa", sdpa)):
    fn(20); torch.cuda.synchronize()
    stop = threading.Event(); out = []
    th = threading.Thread(target=sample, args=(stop, out)); th.start()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    fn(3000); torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / 3000  # wall clock: ours runs on libsip's stream
    stop.set(); th.join()
    cl = np.array([c for c, p in out]); pw = np.array([p for c, p in out])
    print(f"{name}: {tgt.flops/ms/1e9:7.1f} TFLOP/s  sm clock median {np.median(cl):.0f} MHz  power median {np.median(pw):.0f} W  "
          f"-> {tgt.flops/ms/1e9/np.median(cl):.3f} TFLOP/s per MHz", flush=True)
