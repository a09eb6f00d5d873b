"""Tuning targets: the shipped sm_100a cubins plus their device inputs and launch.

* ``gemm``: GEMM+LeakyReLU, C = leaky(A @ B^T), fp16 in/out, fp32 accumulate
  (paper's GEMM workload; config 2 is M=N=K=4096).
* ``attn``: fused attention forward (config 3 is B=4 H=32
  S=4096 D=128).

Device memory is allocated through torch (allocation only); inputs are filled
by libsip's Philox generator (``sip_fill_normal``) and every launch goes
through the evaluator (``sip_measure`` / ``sip_run``) on the cubin words the
search permutes.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from pathlib import Path

from .engine import Launch, get_context

TARGET_DIR = Path(__file__).with_name("targets")
CUBINS = {"gemm": ("gemm_lrelu.cubin", "gemm_lrelu_f16"), "attn": ("attn_fwd.cubin", "attn_fwd_f16")}


def _torch():
    import torch

    if not torch.cuda.is_available():
        from .engine import EngineUnavailable

        raise EngineUnavailable("targets need a CUDA device")
    return torch


@dataclass
class GemmTarget:
    M: int = 4096
    N: int = 4096
    K: int = 4096
    L: int = 1
    slope: float = 0.01
    seed: int = 0
    device: int = 0
    name: str = "gemm"
    _bufs: dict = field(default_factory=dict, repr=False)

    @property
    def flops(self) -> int:
        return 2 * self.M * self.N * self.K * self.L

    @property
    def min_bytes(self) -> int:
        return 2 * self.L * (self.M * self.K + self.N * self.K + self.M * self.N)

    @property
    def out_elems_per_sample(self) -> int:
        return self.M * self.N

    def cubin(self) -> tuple:
        f, func = CUBINS["gemm"]
        return (TARGET_DIR / f).read_bytes(), func

    def allocate(self):
        torch = _torch()
        dev = torch.device("cuda", self.device)
        L, M, N, K = self.L, self.M, self.N, self.K
        self._bufs = {
            "A": torch.empty((L, M, K), dtype=torch.float16, device=dev),
            "B": torch.empty((L, N, K), dtype=torch.float16, device=dev),
            "C": torch.empty((L, M, N), dtype=torch.float16, device=dev),
        }
        self.fill(stream=0)
        return self

    def fill(self, stream: int) -> None:
        """Philox N(0,1) inputs for sample stream `stream` (seeded by self.seed)."""
        ctx = get_context(self.device)
        for i, key in enumerate(("A", "B")):
            t = self._bufs[key]
            ctx.check(ctx.lib.sip_fill_normal(ctx.handle, ctypes.c_void_p(t.data_ptr()), t.numel(), 0,
                                              self.seed * 1000003 + i, stream, 1.0))

    @property
    def inputs(self):
        return self._bufs["A"], self._bufs["B"]

    @property
    def output(self):
        return self._bufs["C"]

    def launch(self, out=None) -> tuple:
        """(Launch struct, params buffer) for the current buffers (output `out` or C)."""
        if not self._bufs:
            self.allocate()
        ctx = get_context(self.device)
        lp = Launch()
        params = ctypes.create_string_buffer(512)
        A, B, C = (self._bufs[k] for k in "ABC")
        if out is not None:
            C = out
        ctx.check(ctx.lib.sip_target_gemm_launch(
            ctx.handle, ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
            ctypes.c_void_p(C.data_ptr()), self.M, self.N, self.K, self.L, ctypes.c_float(self.slope),
            ctypes.byref(lp), params, 512))
        return lp, params

    def reference_output(self):
        """fp32 torch reference of the same op (tests only)."""
        torch = _torch()
        A, B = self.inputs
        y = torch.matmul(A.float(), B.float().transpose(1, 2))
        return torch.where(y > 0, y, y * self.slope)


L2_BYTES = 126 << 20  # B200 L2


def cold_sets(target) -> int:
    """Independent input sets the evaluator rotates through so that no timed launch finds
    its inputs in L2: between two uses of a set the other sets' launches stream at least
    twice the L2 size.  0 means "too many: flush L2 before every timed launch instead"."""
    per = max(1, int(target.min_bytes))
    if per >= 2 * L2_BYTES:
        return 1
    n = -(-2 * L2_BYTES // per) + 1
    return n if n <= 64 else 0


def launch_sets(target, n: int) -> list:
    """[(Launch, params)] of `n` input sets: the target's own buffers, then n - 1 sibling
    targets with their own buffers and Philox streams (kept alive on the target)."""
    from dataclasses import replace

    sets = [target.launch()]
    sibs = getattr(target, "_siblings", [])
    while len(sibs) < n - 1:
        sibs.append(replace(target, seed=target.seed + 7919 * (len(sibs) + 1), _bufs={}).allocate())
    target._siblings = sibs
    sets.extend(t.launch() for t in sibs[: n - 1])
    return sets


TARGET_KINDS = {"gemm": GemmTarget}


def make_target(kind: str, **kw):
    if kind == "attn":
        from .attention import AttnTarget

        return AttnTarget(**kw)
    if kind not in TARGET_KINDS:
        raise ValueError(f"unknown target {kind!r} (want 'gemm' or 'attn')")
    return TARGET_KINDS[kind](**kw)
