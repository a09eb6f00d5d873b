"""Quick GEMM target timing: identity schedule via the evaluator, plus torch matmul for context."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2403_16863_b200.targets import GemmTarget
from paper_2403_16863_b200.evaluator import B200Backend
from paper_2403_16863_b200.cubin import schedule_perm

for (M, N, K) in [(4096, 4096, 4096), (8192, 8192, 8192), (2048, 2048, 2048), (512, 512, 2048)]:
    tgt = GemmTarget(M=M, N=N, K=K).allocate()
    be = B200Backend(tgt, flush_l2=True)
    ident = schedule_perm(be.kernel)
    for flush in (True, False):
        be.flush_l2 = flush
        s = be.measure_perm(ident, reps=20)
        print(f"{M}x{N}x{K} flush={flush}: median {s.value*1e3:.1f} us -> {tgt.flops/s.value/1e9:.1f} TFLOP/s  raw min {min(s.raw)*1e3:.1f}")
    A, B = tgt.inputs
    a, b = A[0], B[0]
    for _ in range(3): torch.matmul(a, b.t())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20): torch.matmul(a, b.t())
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"  torch.matmul fp16: {ms*1e3:.1f} us -> {tgt.flops/ms/1e9:.1f} TFLOP/s")
