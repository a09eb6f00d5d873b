"""Probabilistic verification of a candidate schedule on real hardware (G5/G6).

Semantics follow the reference's differential testing (difftest.py:158-204)
and the paper's 10M-sample check: a *sample* is one
independent random input; the baseline (nvcc) schedule and the candidate run
on it and their outputs are compared.  Here one launch of the target covers
``batch`` samples at once (the targets take a batch dimension), inputs come
from libsip's Philox generator (stream = batch index), and the comparison is
the HBM-bound ``sip_compare`` kernel.  The verdict fails on any element with
|cand - ref| > atol + rtol * |ref|; bit-level differences are counted too
(a pure reordering is expected to be bit-identical).
"""
from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from .backends import MeasurementFailed
from .cubin import Module
from .engine import SIP_E_MEASURE, CmpResult, c_u16p, get_context

# verification shape per target: one sample = one independent problem of this size.
# Shapes are chosen so a batch drives every code path of the target: the GEMM's K=1024
# wraps its 4-stage ring four times per tile and the batch size leaves a partial last
# wave (so the 128x128 half-tile tail runs too, see gemm_batch); the attention head's
# S=512 gives four key blocks, wrapping the 2-stage K/V rings and their phases twice.
VERIFY_SHAPES = {
    "gemm": dict(M=256, N=256, K=1024),
    "attn": dict(B=1, H=1, S=512, D=128),
}
DEFAULT_BATCH = {"gemm": 1024, "attn": 256}


def gemm_batch(sms: int, start: int = 1024) -> int:
    """Largest batch <= start whose 2*L tiles (M=N=256 -> two 128x256 tiles per
    sample) end in a last wave at most half full, so the kernel's half-tile tail runs."""
    for L in range(start, 0, -1):
        tiles = 2 * L
        if tiles > sms and 0 < tiles % sms <= sms // 2:
            return L
    return start
TOLERANCE = {"fp16": (1e-2, 1e-2)}


@dataclass
class VerifyResult:
    samples: int
    passed: int
    failed: int
    first_fail_sample: int
    first_fail_elem: int
    bitdiff_elems: int
    mismatched_elems: int
    max_abs_err: float
    seconds: float
    compared_bytes: int

    @property
    def ok(self) -> bool:
        return self.failed == 0

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k in self.__dataclass_fields__} | {"ok": self.ok}


ATTN_SIGMAS = (0.5, 1.0, 2.0, 4.0)  # input scales attention batches cycle through


class Verifier:
    """Baseline vs candidate over many samples for one target kind."""

    def __init__(self, kind: str, *, device: int = 0, batch: int | None = None, seed: int = 0,
                 shape: dict | None = None):
        from .targets import make_target

        self.kind = kind
        self.ctx = get_context(device)
        self.batch = batch or (gemm_batch(self.ctx.sm_count) if kind == "gemm" else DEFAULT_BATCH[kind])
        sh = dict(VERIFY_SHAPES[kind], **(shape or {}))
        if kind == "gemm":
            self.target = make_target("gemm", L=self.batch, seed=seed, device=device, **sh).allocate()
        else:
            self.target = make_target("attn", seed=seed, device=device, **sh)
            self.target.B *= self.batch
            self.target.allocate()
        cubin, func = self.target.cubin()
        self.module = Module(cubin, func, ctx=self.ctx)
        self.out_ref = self.target.output
        self.out_cand = self.out_ref.clone()
        self.launch_ref, self._p1 = self.target.launch(out=self.out_ref)
        self.launch_cand, self._p2 = self.target.launch(out=self.out_cand)
        self.elems_per_sample = self.out_ref.numel() // self.batch
        self.atol, self.rtol = TOLERANCE["fp16"]
        # attention has a data-dependent path (the lazy O rescale when a row's max grows):
        # batches cycle through input scales so that samples take it in many steps, not
        # only at an item's first; a batch's scale is a function of its index (sharding-safe)
        self.sigmas = ATTN_SIGMAS if kind == "attn" else None

    def _run(self, perm, launch) -> None:
        lib = self.ctx.lib
        p = None if perm is None else np.ascontiguousarray(perm, dtype=np.uint16)
        rc = lib.sip_run(self.module.handle, None if p is None else p.ctypes.data_as(c_u16p),
                         ctypes.byref(launch))
        if rc == SIP_E_MEASURE:
            raise MeasurementFailed(lib.sip_last_error(self.ctx.handle).decode(errors="replace"))
        self.ctx.check(rc)

    def run(self, perm, samples: int, *, first_batch: int = 0, batch_stride: int = 1,
            fail_fast: bool = False, check_every: int = 64) -> VerifyResult:
        """Verify `perm` on batches first_batch, first_batch+stride, ... covering `samples`
        (rounded up to whole batches).  Every batch is enqueued without a host round trip:
        fill (Philox stream = batch index), baseline launch, candidate launch, and an
        accumulating compare; the host synchronises every `check_every` batches (and
        stops early on a failure when `fail_fast`) and once at the end."""
        t0 = time.perf_counter()
        nb = max(1, (samples + self.batch - 1) // self.batch)
        lib = self.ctx.lib
        p = None if perm is None else np.ascontiguousarray(perm, dtype=np.uint16)
        pp = None if p is None else p.ctypes.data_as(c_u16p)
        acc = ctypes.c_void_p()
        self.ctx.check(lib.sip_verify_open(self.ctx.handle, nb * self.batch, self.elems_per_sample,
                                           ctypes.byref(acc)))
        res = CmpResult()
        done = 0
        try:
            for i in range(nb):
                j = first_batch + i * batch_stride
                if self.sigmas:
                    self.target.sigma = self.sigmas[j % len(self.sigmas)]
                self.target.fill(stream=j)
                self._check_run(lib.sip_run_async(self.module.handle, None, ctypes.byref(self.launch_ref)))
                self._check_run(lib.sip_run_async(self.module.handle, pp, ctypes.byref(self.launch_cand)))
                self.ctx.check(lib.sip_verify_compare(
                    acc, ctypes.c_void_p(self.out_ref.data_ptr()), ctypes.c_void_p(self.out_cand.data_ptr()),
                    self.out_ref.numel(), 0, self.atol, self.rtol, j * self.batch))
                done += self.batch
                if (i + 1) % check_every == 0 or i == nb - 1:
                    self._check_run(lib.sip_verify_result(acc, ctypes.byref(res)))
                    if fail_fast and res.failed_samples:
                        break
        finally:
            lib.sip_verify_close(acc)
        dt = time.perf_counter() - t0
        nbytes = 2 * 2 * self.elems_per_sample * done
        failed = int(res.failed_samples)
        return VerifyResult(done, done - failed, failed, int(res.first_fail_sample), int(res.first_fail_elem),
                            int(res.bitdiff_elems), int(res.mismatched_elems), float(res.max_abs_err), dt, nbytes)

    def _check_run(self, rc: int) -> None:
        if rc == SIP_E_MEASURE:
            raise MeasurementFailed(self.ctx.lib.sip_last_error(self.ctx.handle).decode(errors="replace"))
        self.ctx.check(rc)
