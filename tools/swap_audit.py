"""Every single adjacent swap of the identity schedule that involves an extended-class
candidate: legality (reference E, plus hw_safe) and a 64-sample verification of each
hw_safe-legal one.  Prints the failing swaps (legality-model audit on real hardware)."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2403_16863_b200.evaluator import B200Backend
from paper_2403_16863_b200.targets import make_target
from paper_2403_16863_b200.verify import Verifier
from paper_2403_16863_b200.tables import movable_in

kind = sys.argv[1] if len(sys.argv) > 1 else "gemm"
shape = dict(M=512, N=512, K=512) if kind == "gemm" else dict(B=1, H=2, S=512)
tgt = make_target(kind, **shape).allocate()
be = B200Backend(tgt, paired=False)
k = be.kernel
seq = k.schedule
n = len(seq)
tables = be.tables_for(k, "extended")
dk = be.ctx.kernel(tables)
ident = np.arange(n, dtype=np.uint16)
los = [lo for lo in range(n - 1) if movable_in(seq[lo], "extended") or movable_in(seq[lo + 1], "extended")]
legal = dk.legality(np.tile(ident, (len(los), 1)), los, hw_safe=True, min_fixed=be.min_fixed)
ver = Verifier(kind, batch=32)
txt = lambda i: (seq[i].source_text or '').split(';')[0].strip()[10:]
bad = 0
ok_n = 0
for lo, lg in zip(los, legal):
    if not lg:
        continue
    perm = ident.copy()
    perm[lo], perm[lo + 1] = perm[lo + 1], perm[lo]
    vr = ver.run(perm, 64, fail_fast=True, check_every=1)
    if vr.ok:
        ok_n += 1
        print(f"ok   lo={lo}\n    {txt(lo)}\n    {txt(lo + 1)}", flush=True)
        continue
    bad += 1
    print(f"FAIL lo={lo}: maxerr {vr.max_abs_err:.3g}\n    {txt(lo)}\n    {txt(lo + 1)}", flush=True)
print(f"{kind}: {len(los)} candidate slots, {int(legal.sum())} hw_safe-legal swaps, {ok_n} verified, {bad} failed")
