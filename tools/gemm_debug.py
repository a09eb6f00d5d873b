"""One GEMM+LeakyReLU launch at a given shape vs torch fp32 (run under `timeout`)."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2403_16863_b200.evaluator import B200Backend
from paper_2403_16863_b200.targets import GemmTarget

M, N, K, L = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (256, 256, 256, 1)))
tgt = GemmTarget(M=M, N=N, K=K, L=L).allocate()
be = B200Backend(tgt, paired=False)
be.run_perm(None)
torch.cuda.synchronize()
ref = tgt.reference_output()
err = (tgt.output.float() - ref).abs()
tol = 0.05 + 1e-2 * ref.abs()
print(M, N, K, L, "max err", err.max().item(), "ok", bool((err <= tol).all()), flush=True)
