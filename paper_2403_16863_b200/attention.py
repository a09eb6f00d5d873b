"""Attention-forward tuning target (G8): O = softmax(Q K^T * scale) V, fp16 [B, H, S, 128].

The paper's fused-attention workload (BASELINE config 3 is
B=4 H=32 S=4096 D=128, non-causal).  Device memory via torch (allocation only),
inputs from libsip's Philox generator, launches through the evaluator.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

from .engine import Launch, get_context
from .targets import TARGET_DIR, _torch

ATTN_CUBIN = ("attn_fwd.cubin", "attn_fwd_f16")


@dataclass
class AttnTarget:
    B: int = 4
    H: int = 32
    S: int = 4096
    D: int = 128
    seed: int = 0
    device: int = 0
    sigma: float = 0.5
    cubin_file: str = ATTN_CUBIN[0]
    name: str = "attn"
    _bufs: dict = field(default_factory=dict, repr=False)

    @property
    def scale(self) -> float:
        return 1.0 / math.sqrt(self.D)

    @property
    def flops(self) -> int:
        return 4 * self.B * self.H * self.S * self.S * self.D

    @property
    def min_bytes(self) -> int:
        return 4 * 2 * self.B * self.H * self.S * self.D

    def cubin(self) -> tuple:
        return (TARGET_DIR / self.cubin_file).read_bytes(), ATTN_CUBIN[1]

    def allocate(self):
        torch = _torch()
        dev = torch.device("cuda", self.device)
        shape = (self.B, self.H, self.S, self.D)
        self._bufs = {k: torch.empty(shape, dtype=torch.float16, device=dev) for k in "QKVO"}
        self.fill(stream=0)
        return self

    def fill(self, stream: int) -> None:
        ctx = get_context(self.device)
        for i, k in enumerate("QKV"):
            t = self._bufs[k]
            ctx.check(ctx.lib.sip_fill_normal(ctx.handle, ctypes.c_void_p(t.data_ptr()), t.numel(), 0,
                                              self.seed * 1000003 + 17 + i, stream, self.sigma))

    @property
    def inputs(self):
        return tuple(self._bufs[k] for k in "QKV")

    @property
    def output(self):
        return self._bufs["O"]

    def launch(self, out=None) -> tuple:
        if not self._bufs:
            self.allocate()
        ctx = get_context(self.device)
        lp = Launch()
        params = ctypes.create_string_buffer(512)
        Q, K, V, O = (self._bufs[k] for k in "QKVO")
        if out is not None:
            O = out
        ctx.check(ctx.lib.sip_target_attn_launch(
            ctx.handle, ctypes.c_void_p(Q.data_ptr()), ctypes.c_void_p(K.data_ptr()),
            ctypes.c_void_p(V.data_ptr()), ctypes.c_void_p(O.data_ptr()), self.B, self.H, self.S,
            self.D, ctypes.c_float(self.scale), ctypes.byref(lp), params, 512))
        return lp, params

    def reference_output(self):
        """fp32 torch reference (tests only), computed head by head to bound memory."""
        torch = _torch()
        Q, K, V = (t.float() for t in self.inputs)
        out = torch.empty_like(Q)
        for b in range(self.B):
            for h in range(self.H):
                s = (Q[b, h] @ K[b, h].T) * self.scale
                out[b, h] = torch.softmax(s, dim=-1) @ V[b, h]
        return out
