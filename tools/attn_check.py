"""Attention target: correctness of both V-descriptor encodings + timing (exploratory)."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2403_16863_b200.attention import AttnTarget
from paper_2403_16863_b200.evaluator import B200Backend
from paper_2403_16863_b200.cubin import schedule_perm

cubs = ["attn_fwd.cubin"] + sys.argv[1:]
for cub in cubs:
    tgt = AttnTarget(B=1, H=2, S=512, cubin_file=cub).allocate()
    be = B200Backend(tgt)
    be.run_perm(None)
    torch.cuda.synchronize()
    ref = tgt.reference_output()
    err = (tgt.output.float() - ref).abs().max().item()
    print(cub, "max abs err", err, "ref absmax", ref.abs().max().item(), flush=True)
tgt = AttnTarget(B=4, H=32, S=4096).allocate()
be = B200Backend(tgt, flush_l2=False)
s = be.measure_perm(schedule_perm(be.kernel), reps=10)
print(f"attn B4 H32 S4096: {s.value*1e3:.1f} us -> {tgt.flops/s.value/1e9:.1f} TFLOP/s", flush=True)
q, k, v = tgt.inputs
import torch.nn.functional as F
for _ in range(3): F.scaled_dot_product_attention(q, k, v)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(10): F.scaled_dot_product_attention(q, k, v)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"torch sdpa: {ms*1e3:.1f} us -> {tgt.flops/ms/1e9:.1f} TFLOP/s")
