"""Hardware cost backend (G4): real B200 timing of permuted sm_100a cubins.

``B200Backend.measure(kernel, reps)`` keeps the reference contract
(``backends.py:32-39``): the kernel is a (permuted) listing produced by the
cubin frontend; its schedule is turned into a word permutation, the patched
cubin is loaded with ``cuModuleLoadData`` and ``warmup + reps`` launches are
replayed from one CUDA graph with CUDA events around each timed launch
(``sip_measure``).  The value is the median in milliseconds, like the
reference's external protocol (``{"time_ms": x}``, backends.py:25).  Any load
or launch failure raises ``MeasurementFailed``.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .backends import BackendDescriptor, CostSample, MeasurementFailed
from .cubin import Listing, Module, render_listing, schedule_perm
from .engine import SIP_E_MEASURE, EngineError, Launch, c_dblp, c_i32p, c_u16p, get_context
from .ir import Kernel
from .targets import cold_sets, launch_sets, make_target

FIXED_LAT_HEAVY = ("HMMA", "IMMA", "DMMA", "BMMA", "HGMMA", "DFMA", "DADD", "DMUL")


# candidates per sip_measure_round call (big search rounds are split; SIP_ROUND_CHUNK)
ROUND_CHUNK = int(os.environ.get("SIP_ROUND_CHUNK", "64"))

def min_fixed_distance(kernel: Kernel) -> int:
    """Issue distance (cycles) a fixed-latency producer must keep to its consumer
    in hw_safe mode: 8 covers the ALU/FMA/conversion pipes (latency 4-6 on
    Blackwell); listings with legacy tensor or FP64 ops get 40."""
    heavy = any(ins.base_mnemonic in FIXED_LAT_HEAVY for ins in kernel.schedule)
    return 40 if heavy else 8


class B200Backend:
    unit = "ms"
    batched_chains = True  # run_search advances all chains together (driver.py)
    hardware = True        # candidates execute on the GPU: hw_safe legality is enforced

    def __init__(self, target, listing: Listing | None = None, *, device: int = 0, warmup: int = 2,
                 flush_l2: bool = True, paired: bool = True, rounds: bool = True):
        self.target = target
        self.device = device
        self.ctx = get_context(device)
        cubin, func = target.cubin()
        self.listing = listing or render_listing(cubin, func)
        self.module = Module(cubin, func, ctx=self.ctx)
        self.warmup = warmup
        self.flush_l2 = flush_l2
        self.launch, self._params = target.launch()
        self.descriptor = BackendDescriptor(kind="b200", command=func, concurrency_safe=False)
        self.calls = 0
        self.kernel_ms = []  # every timed launch (ms), for roofline accounting
        # paired mode: every candidate is timed against the nvcc schedule inside the same
        # graph; its value is (median cand/ref ratio) x the reference time measured here
        self.paired = paired
        # round mode (measure_batch): one nvcc reference per round of candidates, launches
        # rotated over input sets larger than L2 (targets.cold_sets) instead of a flush
        self.rounds = rounds and paired
        self.nsets = cold_sets(target) if self.rounds else 0
        self._sets = launch_sets(target, self.nsets) if self.nsets else []
        self._set_array = (Launch * max(1, len(self._sets)))(*[lp for lp, _ in self._sets]) if self._sets else None
        self.identity = np.arange(self.listing.n, dtype=np.uint16)
        self.ref_ms = self._measure_single(self.identity, 9).value if paired else None

    @classmethod
    def for_target(cls, kind: str, device: int = 0, **kw):
        tgt = make_target(kind, device=device, **kw).allocate()
        return cls(tgt, device=device)

    @property
    def kernel(self) -> Kernel:
        return self.listing.kernel

    @property
    def min_fixed(self) -> int:
        return min_fixed_distance(self.listing.kernel)

    def tables_for(self, kernel: Kernel, classes: str = "global"):
        """Device tables of `kernel` (a permutation of the listing) with the cubin's
        reuse bits and pinned instructions attached to each identity."""
        from .machine import MachineConfig
        from .tables import KernelTables

        ids = schedule_perm(kernel)
        reuse = [self.listing.reuse[int(i)] for i in ids]
        pinned = [p for p, i in enumerate(ids) if self.listing.pins[int(i)]]
        return KernelTables.build(kernel, MachineConfig(), reuse=reuse, pinned=pinned, classes=classes)

    def perm_of(self, kernel: Kernel) -> np.ndarray:
        return schedule_perm(kernel)

    def measure_perm(self, perm, reps: int = 5) -> CostSample:
        if self.paired:
            ratio, raw = self.ratio(perm, reps)
            return CostSample(ratio * self.ref_ms, self.unit, reps, tuple(r * self.ref_ms for r in raw))
        return self._measure_single(perm, reps)

    def ratio(self, perm, reps: int = 5, ref=None) -> tuple:
        """Median cand/ref time ratio over `reps` interleaved pairs (sip_measure_paired)."""
        perm = np.ascontiguousarray(perm, dtype=np.uint16)
        ref = self.identity if ref is None else np.ascontiguousarray(ref, dtype=np.uint16)
        r_med, ref_med, cand_med = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        raw = np.zeros(reps, dtype=np.float64)
        lib = self.ctx.lib
        rc = lib.sip_measure_paired(self.module.handle, ref.ctypes.data_as(c_u16p),
                                    perm.ctypes.data_as(c_u16p), ctypes.byref(self.launch), self.warmup,
                                    reps, int(self.flush_l2), ctypes.byref(r_med), ctypes.byref(ref_med),
                                    ctypes.byref(cand_med), raw.ctypes.data_as(c_dblp))
        self.calls += 1
        if rc == SIP_E_MEASURE:
            raise MeasurementFailed(lib.sip_last_error(self.ctx.handle).decode(errors="replace"))
        self.ctx.check(rc)
        self.kernel_ms.extend([ref_med.value] * reps + [cand_med.value] * reps)
        return r_med.value, raw.tolist()

    def ratio_round(self, perm, reps: int = 45) -> tuple:
        """Median cand/ref time ratio over `reps` reps of a one-candidate measurement round
        (sip_measure_round): the same protocol that priced the candidate in the search --
        the two schedules alternate (order rotated every rep), launches rotate over cold
        input sets instead of a flush.  Returns (median ratio, per-rep ratios)."""
        if not (self.rounds and self.nsets):
            return self.ratio(perm, reps)
        perm = np.ascontiguousarray(np.asarray(perm, dtype=np.uint16).reshape(1, self.listing.n))
        ratio, refm, candm = (np.zeros(1, dtype=np.float64) for _ in range(3))
        raw = np.zeros((1, reps), dtype=np.float64)
        status = np.zeros(1, dtype=np.int32)
        lib = self.ctx.lib
        rc = lib.sip_measure_round(
            self.module.handle, self.identity.ctypes.data_as(c_u16p), perm.ctypes.data_as(c_u16p), 1,
            self._set_array, len(self._sets), self.warmup, reps, 0,
            ratio.ctypes.data_as(c_dblp), refm.ctypes.data_as(c_dblp), candm.ctypes.data_as(c_dblp),
            raw.ctypes.data_as(c_dblp), status.ctypes.data_as(c_i32p))
        self.calls += 1
        if rc == SIP_E_MEASURE or status[0] != 0:
            raise MeasurementFailed(lib.sip_last_error(self.ctx.handle).decode(errors="replace"))
        self.ctx.check(rc)
        return float(ratio[0]), raw[0].tolist()

    def measure_batch(self, perms, reps: int = 5) -> list:
        """Paired timing of many candidates in one CUDA graph (sip_measure_paired_batch).
        Returns one CostSample per candidate, or a MeasurementFailed instance for a
        candidate whose cubin could not be loaded."""
        perms = np.ascontiguousarray(np.asarray(perms, dtype=np.uint16).reshape(-1, self.listing.n))
        k = perms.shape[0]
        if k == 0:
            return []
        if self.rounds and k > ROUND_CHUNK:
            # a driver holding thousands of modules loads new ones several times slower: big
            # rounds are timed in chunks, each with its own nvcc reference in the rotation and
            # its modules unloaded before the next
            out = []
            for i in range(0, k, ROUND_CHUNK):
                out.extend(self.measure_batch(perms[i:i + ROUND_CHUNK], reps))
            return out
        if not self.paired:
            return [self._try(lambda p=p: self._measure_single(p, reps)) for p in perms]
        ratio, refm, candm = (np.zeros(k, dtype=np.float64) for _ in range(3))
        raw = np.zeros((k, reps), dtype=np.float64)
        status = np.zeros(k, dtype=np.int32)
        lib = self.ctx.lib
        if self.rounds:
            # one reference per round; cold inputs by rotation (nsets > 0) or a flush
            sets, nL = ((self._set_array, len(self._sets)) if self.nsets
                        else (ctypes.pointer(self.launch), 1))
            rc = lib.sip_measure_round(
                self.module.handle, self.identity.ctypes.data_as(c_u16p), perms.ctypes.data_as(c_u16p), k,
                sets, nL, self.warmup, reps, int(self.flush_l2 and not self.nsets),
                ratio.ctypes.data_as(c_dblp), refm.ctypes.data_as(c_dblp), candm.ctypes.data_as(c_dblp),
                raw.ctypes.data_as(c_dblp), status.ctypes.data_as(c_i32p))
        else:
            rc = lib.sip_measure_paired_batch(
                self.module.handle, self.identity.ctypes.data_as(c_u16p), perms.ctypes.data_as(c_u16p), k,
                ctypes.byref(self.launch), self.warmup, reps, int(self.flush_l2), ratio.ctypes.data_as(c_dblp),
                refm.ctypes.data_as(c_dblp), candm.ctypes.data_as(c_dblp), raw.ctypes.data_as(c_dblp),
                status.ctypes.data_as(c_i32p))
        self.calls += k
        if rc == SIP_E_MEASURE:
            raise MeasurementFailed(lib.sip_last_error(self.ctx.handle).decode(errors="replace"))
        self.ctx.check(rc)
        out = []
        if self.rounds and (status == 0).any():
            self.kernel_ms.extend([float(refm[status == 0][0])] * reps)  # the round's one reference
        for i in range(k):
            if status[i] != 0:
                out.append(MeasurementFailed(f"candidate {i}: cubin could not be loaded"))
                continue
            self.kernel_ms.extend(([] if self.rounds else [float(refm[i])] * reps) + [float(candm[i])] * reps)
            out.append(CostSample(float(ratio[i]) * self.ref_ms, self.unit, reps,
                                  tuple(float(r) * self.ref_ms for r in raw[i])))
        return out

    @staticmethod
    def _try(fn):
        try:
            return fn()
        except MeasurementFailed as exc:
            return exc

    def _measure_single(self, perm, reps: int = 5) -> CostSample:
        perm = np.ascontiguousarray(perm, dtype=np.uint16)
        med = ctypes.c_double()
        raw = np.zeros(reps, dtype=np.float64)
        lib = self.ctx.lib
        rc = lib.sip_measure(self.module.handle, perm.ctypes.data_as(c_u16p), ctypes.byref(self.launch),
                             self.warmup, reps, int(self.flush_l2), ctypes.byref(med),
                             raw.ctypes.data_as(c_dblp))
        self.calls += 1
        if rc == SIP_E_MEASURE:
            raise MeasurementFailed(lib.sip_last_error(self.ctx.handle).decode(errors="replace"))
        self.ctx.check(rc)
        self.kernel_ms.extend(raw.tolist())
        return CostSample(med.value, self.unit, reps, tuple(raw.tolist()))

    def measure(self, kernel: Kernel, reps: int = 5) -> CostSample:
        if len(kernel.schedule) != self.listing.n:
            raise MeasurementFailed("schedule does not match the loaded cubin")
        try:
            perm = self.perm_of(kernel)
        except ValueError as exc:
            raise MeasurementFailed(f"schedule is not a listing of the loaded cubin: {exc}") from None
        if not np.array_equal(np.sort(perm), self.identity):
            raise MeasurementFailed("schedule is not a permutation of the loaded cubin's instructions")
        return self.measure_perm(perm, reps)

    def run_perm(self, perm) -> None:
        perm = None if perm is None else np.ascontiguousarray(perm, dtype=np.uint16)
        lib = self.ctx.lib
        rc = lib.sip_run(self.module.handle, None if perm is None else perm.ctypes.data_as(c_u16p),
                         ctypes.byref(self.launch))
        if rc == SIP_E_MEASURE:
            raise MeasurementFailed(lib.sip_last_error(self.ctx.handle).decode(errors="replace"))
        self.ctx.check(rc)
