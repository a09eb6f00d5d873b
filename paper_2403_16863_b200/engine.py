"""ctypes binding of libsip.so (include/sip.h) -- the only path to the device.

There is no CPU fallback: if the shared library or a CUDA device is missing,
every entry point raises ``EngineUnavailable`` with the reason.
"""
from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from .tables import MAX_REFS, KernelTables

LIB_PATH = Path(__file__).with_name("libsip.so")

SIP_OK, SIP_E_ARG, SIP_E_CUDA, SIP_E_MEASURE, SIP_E_NOCAND, SIP_E_ELF, SIP_E_STATE = range(7)
ST_ACCEPTED, ST_PRICED, ST_BOUNDARY, ST_DEPENDENCY, ST_TEST, ST_MEASURE, ST_HWSAFE = range(7)
STATUS_REASON = {ST_BOUNDARY: "boundary", ST_DEPENDENCY: "dependency", ST_TEST: "test-failure",
                 ST_MEASURE: "measurement", ST_HWSAFE: "hw-safety"}

c_u16p = ctypes.POINTER(ctypes.c_uint16)
c_u8p = ctypes.POINTER(ctypes.c_uint8)
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_u32p = ctypes.POINTER(ctypes.c_uint32)
c_u64p = ctypes.POINTER(ctypes.c_uint64)
c_dblp = ctypes.POINTER(ctypes.c_double)


class EngineUnavailable(RuntimeError):
    """libsip.so or the B200 it drives is not available."""


class EngineError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = code
        super().__init__(f"libsip error {code}: {msg}")


class Tables(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32), ("words", ctypes.c_int32),
        ("ctrl", c_u32p), ("lat", c_u32p), ("klass", c_u8p),
        ("reads", c_u64p), ("writes", c_u64p), ("refs", ctypes.c_void_p),
        ("nrefs", c_u8p), ("cut", c_u8p), ("pin", c_u8p), ("guard", c_u64p),
    ]


class AnnealCfg(ctypes.Structure):
    _fields_ = [("budget", ctypes.c_int32), ("unsafe_moves", ctypes.c_int32),
                ("hw_safe", ctypes.c_int32), ("min_fixed_distance", ctypes.c_int32),
                ("temperature", c_dblp)]


RECORD_DTYPE = np.dtype([("time", "<f8"), ("lo", "<i4"), ("candidate", "<u2"),
                         ("direction", "u1"), ("status", "u1")])
SUMMARY_DTYPE = np.dtype([("t0", "<f8"), ("best_energy", "<f8"), ("current_energy", "<f8"),
                          ("best_iter", "<i4"), ("ambiguous", "<i4"), ("replayed", "<i8"),
                          ("priced", "<i4"), ("pad", "<i4")])


class EpochResult(ctypes.Structure):
    _fields_ = [("champion_chain", ctypes.c_int32), ("pad", ctypes.c_int32), ("best_energy", ctypes.c_double),
                ("best_seed", ctypes.c_int64), ("priced", ctypes.c_int64), ("replayed", ctypes.c_int64),
                ("ambiguous", ctypes.c_int64)]


class Launch(ctypes.Structure):
    _fields_ = [("grid", ctypes.c_uint32 * 3), ("block", ctypes.c_uint32 * 3),
                ("cluster", ctypes.c_uint32 * 3), ("smem_bytes", ctypes.c_uint32),
                ("params", ctypes.c_void_p), ("param_offsets", ctypes.c_void_p),
                ("nparams", ctypes.c_uint32), ("params_size", ctypes.c_uint32)]


class CmpResult(ctypes.Structure):
    _fields_ = [("checked_elems", ctypes.c_int64), ("mismatched_elems", ctypes.c_int64),
                ("bitdiff_elems", ctypes.c_int64), ("failed_samples", ctypes.c_int64),
                ("first_fail_sample", ctypes.c_int64), ("first_fail_elem", ctypes.c_int64),
                ("max_abs_err", ctypes.c_double)]


def _ptr(arr: np.ndarray, ctype):
    return arr.ctypes.data_as(ctype)


_SIGS = {
    "sip_version": ([], ctypes.c_char_p),
    "sip_device_count": ([c_i32p], ctypes.c_int),
    "sip_open": ([ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "sip_close": ([ctypes.c_void_p], ctypes.c_int),
    "sip_last_error": ([ctypes.c_void_p], ctypes.c_char_p),
    "sip_kernel_create": ([ctypes.c_void_p, ctypes.POINTER(Tables), ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "sip_kernel_destroy": ([ctypes.c_void_p], ctypes.c_int),
    "sip_kernel_candidates": ([ctypes.c_void_p, c_i32p], ctypes.c_int),
    "sip_legality_rows": ([ctypes.c_void_p, c_u32p, c_u32p], ctypes.c_int),
    "sip_legality_query": ([ctypes.c_void_p, c_u16p, c_i32p, ctypes.c_int32, ctypes.c_int32,
                            ctypes.c_int32, c_u8p], ctypes.c_int),
    "sip_simulate": ([ctypes.c_void_p, c_u16p, ctypes.c_int32, c_i64p, c_i32p,
                      ctypes.POINTER(ctypes.c_int8)], ctypes.c_int),
    "sip_anneal": ([ctypes.c_void_p, ctypes.POINTER(AnnealCfg), c_i64p, ctypes.c_int32,
                    ctypes.c_void_p, c_u16p, c_u16p, ctypes.c_void_p], ctypes.c_int),
    "sip_anneal_ex": ([ctypes.c_void_p, ctypes.POINTER(AnnealCfg), c_i64p, ctypes.c_int32, c_u16p,
                       ctypes.c_void_p, c_u16p, c_u16p, ctypes.c_void_p, c_u16p, c_i32p], ctypes.c_int),
    "sip_anneal_epoch": ([ctypes.c_void_p, ctypes.POINTER(AnnealCfg), ctypes.c_int64, ctypes.c_int32, c_u16p,
                          ctypes.c_void_p, c_u16p], ctypes.c_int),
    "sip_anneal_keep": ([ctypes.c_void_p, ctypes.POINTER(AnnealCfg), c_i64p, ctypes.c_int32, c_u16p,
                         ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "sip_results_fetch": ([ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, c_u16p, c_u16p],
                          ctypes.c_int),
    "sip_results_destroy": ([ctypes.c_void_p], ctypes.c_int),
    "sip_anneal_keep_reduced": ([ctypes.c_void_p, ctypes.POINTER(AnnealCfg), c_i64p, ctypes.c_int64,
                                 ctypes.c_int32, c_u16p, ctypes.POINTER(EpochResult),
                                 ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "sip_results_summary": ([ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p], ctypes.c_int),
    "sip_anneal_wave": ([ctypes.c_void_p, c_i32p], ctypes.c_int),
    "sip_anneal_state_bytes": ([ctypes.c_void_p, ctypes.c_int32, c_i64p], ctypes.c_int),
    "sip_host_alloc": ([ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "sip_host_free": ([ctypes.c_void_p], ctypes.c_int),
    "sip_chains_create": ([ctypes.c_void_p, ctypes.POINTER(AnnealCfg), c_i64p, c_dblp,
                           ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "sip_chains_propose": ([ctypes.c_void_p, c_i32p, c_u16p], ctypes.c_int),
    "sip_chains_resolve": ([ctypes.c_void_p, c_dblp, c_u8p], ctypes.c_int),
    "sip_chains_adopt": ([ctypes.c_void_p, c_u16p, ctypes.c_double, ctypes.c_double], ctypes.c_int),
    "sip_chains_result": ([ctypes.c_void_p, ctypes.c_void_p, c_u16p, c_u16p, ctypes.c_void_p], ctypes.c_int),
    "sip_chains_destroy": ([ctypes.c_void_p], ctypes.c_int),
    "sip_module_open": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_char_p,
                         ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "sip_module_close": ([ctypes.c_void_p], ctypes.c_int),
    "sip_module_info": ([ctypes.c_void_p, c_i32p, c_u64p], ctypes.c_int),
    "sip_module_words": ([ctypes.c_void_p, c_u64p], ctypes.c_int),
    "sip_module_pins": ([ctypes.c_void_p, c_u8p], ctypes.c_int),
    "sip_module_patch": ([ctypes.c_void_p, c_u16p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "sip_measure": ([ctypes.c_void_p, c_u16p, ctypes.POINTER(Launch), ctypes.c_int32, ctypes.c_int32,
                     ctypes.c_int32, c_dblp, c_dblp], ctypes.c_int),
    "sip_measure_paired": ([ctypes.c_void_p, c_u16p, c_u16p, ctypes.POINTER(Launch), ctypes.c_int32,
                            ctypes.c_int32, ctypes.c_int32, c_dblp, c_dblp, c_dblp, c_dblp], ctypes.c_int),
    "sip_measure_paired_batch": ([ctypes.c_void_p, c_u16p, c_u16p, ctypes.c_int32, ctypes.POINTER(Launch),
                                  ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, c_dblp, c_dblp, c_dblp,
                                  c_dblp, c_i32p], ctypes.c_int),
    "sip_measure_round": ([ctypes.c_void_p, c_u16p, c_u16p, ctypes.c_int32, ctypes.POINTER(Launch),
                           ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, c_dblp, c_dblp,
                           c_dblp, c_dblp, c_i32p], ctypes.c_int),
    "sip_run": ([ctypes.c_void_p, c_u16p, ctypes.POINTER(Launch)], ctypes.c_int),
    "sip_run_async": ([ctypes.c_void_p, c_u16p, ctypes.POINTER(Launch)], ctypes.c_int),
    "sip_verify_open": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p)],
                        ctypes.c_int),
    "sip_verify_compare": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32,
                            ctypes.c_double, ctypes.c_double, ctypes.c_int64], ctypes.c_int),
    "sip_verify_result": ([ctypes.c_void_p, ctypes.POINTER(CmpResult)], ctypes.c_int),
    "sip_verify_close": ([ctypes.c_void_p], ctypes.c_int),
    "sip_fill_normal": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32,
                         ctypes.c_uint64, ctypes.c_uint64, ctypes.c_float], ctypes.c_int),
    "sip_compare": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32,
                     ctypes.c_double, ctypes.c_double, ctypes.c_int64, ctypes.c_int64,
                     ctypes.POINTER(CmpResult)], ctypes.c_int),
    "sip_sample_inputs": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                           c_i32p, c_i32p, c_i32p, c_u8p], ctypes.c_int),
    "sip_sample_inputs_device": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                  ctypes.c_int32, c_i32p, c_i32p, c_i32p, ctypes.c_void_p], ctypes.c_int),
    "sip_vm_exec": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, c_i64p, c_i32p, c_i32p,
                     ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, c_i32p,
                     c_i64p], ctypes.c_int),
    "sip_vm_cell_diff": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                          ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, c_i32p], ctypes.c_int),
    "sip_target_gemm_launch": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                ctypes.c_float, ctypes.POINTER(Launch), ctypes.c_void_p,
                                ctypes.c_uint32], ctypes.c_int),
    "sip_target_attn_launch": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                ctypes.c_int32, ctypes.c_float, ctypes.POINTER(Launch),
                                ctypes.c_void_p, ctypes.c_uint32], ctypes.c_int),
    "sip_comm_unique_id": ([c_u8p], ctypes.c_int),
    "sip_comm_create": ([ctypes.c_void_p, c_u8p, ctypes.c_int32, ctypes.c_int32,
                         ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "sip_comm_destroy": ([ctypes.c_void_p], ctypes.c_int),
    "sip_nccl_exchange": ([ctypes.c_void_p, ctypes.c_void_p, c_u16p, ctypes.c_int32, ctypes.c_void_p,
                           ctypes.c_void_p, c_u16p], ctypes.c_int),
    "sip_comm_allreduce": ([ctypes.c_void_p, c_dblp, ctypes.c_int32, ctypes.c_int32], ctypes.c_int),
    "sip_comm_barrier": ([ctypes.c_void_p], ctypes.c_int),
}

_lib = None
_lib_lock = threading.Lock()


def load_library(path: Path | None = None) -> ctypes.CDLL:
    """Load libsip.so and bind every C-ABI symbol (raises if any is missing)."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path or os.environ.get("SIP_LIB", LIB_PATH))
        if not p.exists():
            raise EngineUnavailable(f"{p} not built (run __graft_entry__.build())")
        lib = ctypes.CDLL(str(p))
        missing = []
        for name, (argtypes, restype) in _SIGS.items():
            try:
                fn = getattr(lib, name)
            except AttributeError:
                missing.append(name)
                continue
            fn.argtypes = argtypes
            fn.restype = restype
        lib.sip_missing = tuple(missing)
        if path is None:
            _lib = lib
        return lib


class Context:
    """One device context (sip_ctx); one per GPU and host thread."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        count = ctypes.c_int32(0)
        self.lib.sip_device_count(ctypes.byref(count))
        if count.value < 1:
            raise EngineUnavailable("no CUDA device visible; the SIP engine has no CPU fallback")
        h = ctypes.c_void_p()
        rc = self.lib.sip_open(device, ctypes.byref(h))
        if rc != SIP_OK:
            raise EngineUnavailable(f"sip_open({device}) failed with code {rc} (needs an sm_100 GPU)")
        self.handle = h
        self.device = device
        self._kernels: dict = {}
        self._sm_count = None

    @property
    def sm_count(self) -> int:
        if self._sm_count is None:
            import torch

            self._sm_count = int(torch.cuda.get_device_properties(self.device).multi_processor_count)
        return self._sm_count

    def check(self, rc: int) -> None:
        if rc != SIP_OK:
            msg = self.lib.sip_last_error(self.handle).decode(errors="replace")
            raise EngineError(rc, msg)

    def kernel(self, tables: KernelTables) -> "DeviceKernel":
        key = (id(tables),)
        dk = self._kernels.get(key)
        if dk is None or dk.tables is not tables:
            dk = DeviceKernel(self, tables)
            self._kernels = {key: dk}  # keep only the latest listing resident
        return dk

    def close(self) -> None:
        if getattr(self, "handle", None):
            self._kernels.clear()
            self.lib.sip_close(self.handle)
            self.handle = None


_contexts: dict = {}


def get_context(device: int | None = None) -> Context:
    dev = int(os.environ.get("SIP_DEVICE", "0")) if device is None else device
    ctx = _contexts.get(dev)
    if ctx is None:
        ctx = Context(dev)
        _contexts[dev] = ctx
    return ctx


def temperature_schedule(t_max: float, cooling: float, budget: int) -> np.ndarray:
    """T at the start of each iteration: repeated IEEE division (anneal.py:176-202)."""
    out = np.empty(budget, dtype=np.float64)
    t = t_max
    for i in range(budget):
        out[i] = t
        t /= cooling
    return out


class DeviceKernel:
    """Device-resident tables of one listing plus its G1 legality rows."""

    def __init__(self, ctx: Context, tables: KernelTables):
        self.ctx = ctx
        self.tables = tables
        self.n = tables.n
        self._keep = [tables.ctrl, tables.lat, tables.klass, tables.reads, tables.writes,
                      tables.refs, tables.nrefs, tables.cut, tables.pin, tables.guard]
        guard = None if tables.guard is None else np.ascontiguousarray(tables.guard.reshape(-1))
        self._keep.append(guard)
        t = Tables(
            tables.n, tables.words,
            _ptr(tables.ctrl, c_u32p), _ptr(tables.lat, c_u32p), _ptr(tables.klass, c_u8p),
            _ptr(tables.reads, c_u64p), _ptr(tables.writes, c_u64p),
            tables.refs.ctypes.data_as(ctypes.c_void_p),
            _ptr(tables.nrefs, c_u8p), _ptr(tables.cut, c_u8p), _ptr(tables.pin, c_u8p),
            None if guard is None else _ptr(guard, c_u64p),
        )
        h = ctypes.c_void_p()
        ctx.check(ctx.lib.sip_kernel_create(ctx.handle, ctypes.byref(t), ctypes.byref(h)))
        self.handle = h
        k = ctypes.c_int32()
        ctx.check(ctx.lib.sip_kernel_candidates(h, ctypes.byref(k)))
        self.k = k.value

    def __del__(self):
        try:
            if self.handle:
                self.ctx.lib.sip_kernel_destroy(self.handle)
        except Exception:
            pass

    def legality_rows(self):
        nw = (self.n + 31) // 32
        after = np.zeros((max(self.k, 1), nw), dtype=np.uint32)
        before = np.zeros_like(after)
        self.ctx.check(self.ctx.lib.sip_legality_rows(self.handle, _ptr(after, c_u32p),
                                                      _ptr(before, c_u32p)))
        return after[: self.k], before[: self.k]

    def legality(self, scheds, los, hw_safe: bool = False, min_fixed: int = 0) -> np.ndarray:
        s = np.ascontiguousarray(np.asarray(scheds, dtype=np.uint16).reshape(-1, self.n))
        lo = np.ascontiguousarray(np.asarray(los, dtype=np.int32))
        out = np.zeros(len(lo), dtype=np.uint8)
        self.ctx.check(self.ctx.lib.sip_legality_query(self.handle, _ptr(s, c_u16p), _ptr(lo, c_i32p),
                                                       len(lo), int(hw_safe), int(min_fixed),
                                                       _ptr(out, c_u8p)))
        return out

    def simulate(self, scheds, detail: bool = False):
        s = np.ascontiguousarray(np.asarray(scheds, dtype=np.uint16).reshape(-1, self.n))
        cnt = s.shape[0]
        totals = np.zeros(cnt, dtype=np.int64)
        waited = binding = None
        wp = bp = None
        if detail:
            waited = np.zeros((cnt, self.n), dtype=np.int32)
            binding = np.zeros((cnt, self.n), dtype=np.int8)
            wp, bp = _ptr(waited, c_i32p), binding.ctypes.data_as(ctypes.POINTER(ctypes.c_int8))
        self.ctx.check(self.ctx.lib.sip_simulate(self.handle, _ptr(s, c_u16p), cnt,
                                                 _ptr(totals, c_i64p), wp, bp))
        return (totals, waited, binding) if detail else totals

    def _cfg(self, temps: np.ndarray, unsafe: bool, hw_safe: bool, min_fixed: int) -> AnnealCfg:
        return AnnealCfg(len(temps), int(unsafe), int(hw_safe), int(min_fixed), _ptr(temps, c_dblp))

    def anneal(self, seeds, temps: np.ndarray, unsafe: bool = False, hw_safe: bool = False,
               min_fixed: int = 0, want_schedules: bool = True):
        """Fused simulator-energy chains (sip_anneal).  Returns (history, best, current, summary)."""
        seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.int64))
        temps = np.ascontiguousarray(temps, dtype=np.float64)
        C, B = len(seeds), len(temps)
        hist = np.zeros((C, B), dtype=RECORD_DTYPE)
        summ = np.zeros(C, dtype=SUMMARY_DTYPE)
        best = cur = None
        bp = cp = None
        if want_schedules:
            best = np.zeros((C, self.n), dtype=np.uint16)
            cur = np.zeros((C, self.n), dtype=np.uint16)
            bp, cp = _ptr(best, c_u16p), _ptr(cur, c_u16p)
        cfg = self._cfg(temps, unsafe, hw_safe, min_fixed)
        self.ctx.check(self.ctx.lib.sip_anneal(self.handle, ctypes.byref(cfg), _ptr(seeds, c_i64p), C,
                                               hist.ctypes.data_as(ctypes.c_void_p), bp, cp,
                                               summ.ctypes.data_as(ctypes.c_void_p)))
        return hist, best, cur, summ

    def anneal_epoch(self, seeds, temps: np.ndarray, start=None, unsafe: bool = False,
                     with_history: bool = True):
        """Fused chains from `start` (identity if None); returns (history|None, summary,
        champion schedule, champion chain).  Schedules of other chains stay on the device."""
        seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.int64))
        temps = np.ascontiguousarray(temps, dtype=np.float64)
        C, B = len(seeds), len(temps)
        hist = np.zeros((C, B), dtype=RECORD_DTYPE) if with_history else None
        summ = np.zeros(C, dtype=SUMMARY_DTYPE)
        champ = np.zeros(self.n, dtype=np.uint16)
        wch = ctypes.c_int32(-1)
        st = None if start is None else np.ascontiguousarray(start, dtype=np.uint16)
        cfg = self._cfg(temps, unsafe, False, 0)
        self.ctx.check(self.ctx.lib.sip_anneal_ex(
            self.handle, ctypes.byref(cfg), _ptr(seeds, c_i64p), C,
            None if st is None else _ptr(st, c_u16p),
            None if hist is None else hist.ctypes.data_as(ctypes.c_void_p), None, None,
            summ.ctypes.data_as(ctypes.c_void_p), _ptr(champ, c_u16p), ctypes.byref(wch)))
        return hist, summ, champ, wch.value

    def anneal_epoch_reduced(self, seed_base: int, chains: int, temps: np.ndarray, start=None,
                             unsafe: bool = False):
        """One sharded-search epoch (sip_anneal_epoch): `chains` fused chains with seeds
        seed_base + c generated on the device, reduced there to the champion under
        driver.py:81-85's ranking plus instrumentation sums.  Returns (dict, schedule)."""
        temps = np.ascontiguousarray(temps, dtype=np.float64)
        champ = np.zeros(self.n, dtype=np.uint16)
        st = None if start is None else np.ascontiguousarray(start, dtype=np.uint16)
        res = EpochResult()
        cfg = self._cfg(temps, unsafe, False, 0)
        self.ctx.check(self.ctx.lib.sip_anneal_epoch(
            self.handle, ctypes.byref(cfg), int(seed_base), int(chains),
            None if st is None else _ptr(st, c_u16p), ctypes.byref(res), _ptr(champ, c_u16p)))
        out = {f: getattr(res, f) for f, _ in EpochResult._fields_ if f != "pad"}
        return out, champ

    def wave_chains(self) -> int:
        """Chains filling every SM once with the fused kernel (sip_anneal_wave)."""
        v = ctypes.c_int32()
        self.ctx.check(self.ctx.lib.sip_anneal_wave(self.handle, ctypes.byref(v)))
        return int(v.value)

    def state_bytes(self, budget: int) -> int:
        """HBM bytes one fused chain keeps (sip_anneal_state_bytes)."""
        v = ctypes.c_int64()
        self.ctx.check(self.ctx.lib.sip_anneal_state_bytes(self.handle, int(budget), ctypes.byref(v)))
        return int(v.value)

    def anneal_keep(self, seeds, temps: np.ndarray, start=None, unsafe: bool = False,
                    hw_safe: bool = False, min_fixed: int = 0):
        """Fused chains whose histories and schedules stay on the device (sip_anneal_keep)."""
        seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.int64))
        temps = np.ascontiguousarray(temps, dtype=np.float64)
        C = len(seeds)
        summ = pinned_pool(self.ctx.lib).records(C, SUMMARY_DTYPE)
        st = None if start is None else np.ascontiguousarray(start, dtype=np.uint16)
        cfg = self._cfg(temps, unsafe, hw_safe, min_fixed)
        h = ctypes.c_void_p()
        self.ctx.check(self.ctx.lib.sip_anneal_keep(
            self.handle, ctypes.byref(cfg), _ptr(seeds, c_i64p), C,
            None if st is None else _ptr(st, c_u16p), summ.ctypes.data_as(ctypes.c_void_p), ctypes.byref(h)))
        return summ, DeviceResults(self, h, C, len(temps))

    def anneal_keep_reduced(self, seeds, temps: np.ndarray, start=None, unsafe: bool = False,
                            hw_safe: bool = False, min_fixed: int = 0):
        """Fused chains left entirely in HBM (sip_anneal_keep_reduced): only the device-reduced
        champion and sums come back; consecutive seeds are generated on the device.
        Returns (EpochResult dict, DeviceResults)."""
        if isinstance(seeds, range) and seeds.step == 1:
            # run_search's consecutive seeds (driver.py:73-79) as a range: nothing per chain
            # on the host (an int64 array of 227 k seeds and its np.diff check cost ~0.5 ms
            # a step); the device generates them
            C, consecutive, base = len(seeds), True, seeds.start
        else:
            seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.int64))
            C = len(seeds)
            consecutive = C > 0 and (C == 1 or bool(np.all(np.diff(seeds) == 1)))
            base = int(seeds[0]) if consecutive else 0
        temps = np.ascontiguousarray(temps, dtype=np.float64)
        st = None if start is None else np.ascontiguousarray(start, dtype=np.uint16)
        cfg = self._cfg(temps, unsafe, hw_safe, min_fixed)
        res = EpochResult()
        h = ctypes.c_void_p()
        self.ctx.check(self.ctx.lib.sip_anneal_keep_reduced(
            self.handle, ctypes.byref(cfg), None if consecutive else _ptr(seeds, c_i64p),
            base, C, None if st is None else _ptr(st, c_u16p), ctypes.byref(res), ctypes.byref(h)))
        out = {f: getattr(res, f) for f, _ in EpochResult._fields_ if f != "pad"}
        return out, DeviceResults(self, h, C, len(temps))

    def chains(self, seeds, t0, temps: np.ndarray, unsafe: bool = False, hw_safe: bool = False,
               min_fixed: int = 0) -> "StepChains":
        return StepChains(self, seeds, t0, temps, unsafe, hw_safe, min_fixed)


class _PinnedPool:
    """Page-locked host blocks (sip_host_alloc) for results the device writes whole, such
    as the per-chain summaries: the copy runs at full DMA rate with no first-touch page
    faults.  A block returns to the pool when the last array viewing it is dropped."""

    def __init__(self, lib):
        self.lib = lib
        self.free: dict = {}  # nbytes -> [addresses]
        self.lock = threading.Lock()
        self.allocated = 0  # blocks obtained from sip_host_alloc (never returned to CUDA)

    def records(self, count: int, dtype) -> np.ndarray:
        dtype = np.dtype(dtype)
        nbytes = max(1, count * dtype.itemsize)
        with self.lock:
            blocks = self.free.get(nbytes)
            addr = blocks.pop() if blocks else None
        if addr is None:
            p = ctypes.c_void_p()
            if self.lib.sip_host_alloc(nbytes, ctypes.byref(p)) != 0 or not p.value:
                return np.zeros(count, dtype=dtype)  # pageable memory still works
            addr = p.value
            self.allocated += 1
        raw = (ctypes.c_char * nbytes).from_address(addr)
        raw._block = _PinnedBlock(self, nbytes, addr)  # every view of the array keeps raw alive
        return np.frombuffer(raw, dtype=np.uint8, count=count * dtype.itemsize).view(dtype)

    def release(self, nbytes: int, addr: int) -> None:
        with self.lock:
            self.free.setdefault(nbytes, []).append(addr)


_POOL: _PinnedPool | None = None


def pinned_pool(lib) -> _PinnedPool:
    """The process-wide pool (blocks are portable across the per-GPU contexts)."""
    global _POOL
    if _POOL is None:
        _POOL = _PinnedPool(lib)
    return _POOL


class _PinnedBlock:
    def __init__(self, pool: _PinnedPool, nbytes: int, addr: int):
        self.pool, self.nbytes, self.addr = pool, nbytes, addr

    def __del__(self):
        self.pool.release(self.nbytes, self.addr)


class DeviceResults:
    """Per-chain histories and schedules left in HBM by sip_anneal_keep; fetched on demand."""

    def __init__(self, dk: DeviceKernel, handle, chains: int, budget: int):
        self.dk = dk  # keeps the listing (and its workspace) alive
        self.handle = handle
        self.C = chains
        self.budget = budget
        self._cache: dict = {}

    def summary(self, first: int = 0, count: int | None = None) -> np.ndarray:
        """Per-chain summaries [first, first + count) (sip_results_summary)."""
        count = self.C - first if count is None else count
        out = pinned_pool(self.dk.ctx.lib).records(count, SUMMARY_DTYPE)
        ctx = self.dk.ctx
        ctx.check(ctx.lib.sip_results_summary(self.handle, first, count, out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def fetch(self, c: int):
        """(records[budget], best[n], current[n]) of chain c."""
        hit = self._cache.get(c)
        if hit is not None:
            return hit
        n = self.dk.n
        hist = np.zeros(self.budget, dtype=RECORD_DTYPE)
        best = np.zeros(n, dtype=np.uint16)
        cur = np.zeros(n, dtype=np.uint16)
        ctx = self.dk.ctx
        ctx.check(ctx.lib.sip_results_fetch(self.handle, c, 1, hist.ctypes.data_as(ctypes.c_void_p),
                                            _ptr(best, c_u16p), _ptr(cur, c_u16p)))
        self._cache[c] = (hist, best, cur)
        return self._cache[c]

    def __del__(self):
        try:
            if self.handle:
                self.dk.ctx.lib.sip_results_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


class StepChains:
    """Step-mode chains: the device proposes, the host prices (any backend)."""

    def __init__(self, dk: DeviceKernel, seeds, t0, temps, unsafe, hw_safe, min_fixed):
        self.dk = dk
        ctx = dk.ctx
        self.seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.int64))
        self.C = len(self.seeds)
        self.t0 = np.ascontiguousarray(np.asarray(t0, dtype=np.float64).reshape(self.C))
        self.temps = np.ascontiguousarray(temps, dtype=np.float64)
        cfg = dk._cfg(self.temps, unsafe, hw_safe, min_fixed)
        h = ctypes.c_void_p()
        ctx.check(ctx.lib.sip_chains_create(dk.handle, ctypes.byref(cfg), _ptr(self.seeds, c_i64p),
                                            _ptr(self.t0, c_dblp), self.C, ctypes.byref(h)))
        self.handle = h
        self.lo = np.zeros(self.C, dtype=np.int32)
        self.cand = np.zeros((self.C, dk.n), dtype=np.uint16)

    def propose(self, with_schedules: bool = True):
        ctx = self.dk.ctx
        sp = _ptr(self.cand, c_u16p) if with_schedules else None
        ctx.check(ctx.lib.sip_chains_propose(self.handle, _ptr(self.lo, c_i32p), sp))
        return self.lo, self.cand

    def resolve(self, times, status) -> None:
        t = np.ascontiguousarray(np.asarray(times, dtype=np.float64))
        s = np.ascontiguousarray(np.asarray(status, dtype=np.uint8))
        ctx = self.dk.ctx
        ctx.check(ctx.lib.sip_chains_resolve(self.handle, _ptr(t, c_dblp), _ptr(s, c_u8p)))

    def adopt(self, sched, energy: float, time: float) -> None:
        s = np.ascontiguousarray(np.asarray(sched, dtype=np.uint16))
        ctx = self.dk.ctx
        ctx.check(ctx.lib.sip_chains_adopt(self.handle, _ptr(s, c_u16p), float(energy), float(time)))

    def result(self):
        C, B, n = self.C, len(self.temps), self.dk.n
        hist = np.zeros((C, B), dtype=RECORD_DTYPE)
        summ = np.zeros(C, dtype=SUMMARY_DTYPE)
        best = np.zeros((C, n), dtype=np.uint16)
        cur = np.zeros((C, n), dtype=np.uint16)
        ctx = self.dk.ctx
        ctx.check(ctx.lib.sip_chains_result(self.handle, hist.ctypes.data_as(ctypes.c_void_p),
                                            _ptr(best, c_u16p), _ptr(cur, c_u16p),
                                            summ.ctypes.data_as(ctypes.c_void_p)))
        return hist, best, cur, summ

    def __del__(self):
        try:
            if self.handle:
                self.dk.ctx.lib.sip_chains_destroy(self.handle)
        except Exception:
            pass


__all__ = ["Context", "DeviceKernel", "StepChains", "EngineUnavailable", "EngineError",
           "get_context", "load_library", "temperature_schedule", "KernelTables", "MAX_REFS",
           "RECORD_DTYPE", "SUMMARY_DTYPE", "Launch", "CmpResult", "STATUS_REASON"]
