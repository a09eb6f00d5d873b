"""ctypes wrapper of the CPU oracle (oracle/sip_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product
package.  Every function is a restatement of the reference algorithm cited in
sip_oracle.c and is pinned against tests/golden/reference.json.gz.
"""
from __future__ import annotations

import ctypes
import json
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libsip_oracle.so"

RECORD_DTYPE = np.dtype([("time", "<f8"), ("lo", "<i4"), ("candidate", "<u2"),
                         ("direction", "u1"), ("status", "u1")])
SUMMARY_DTYPE = np.dtype([("t0", "<f8"), ("best_energy", "<f8"), ("current_energy", "<f8"),
                          ("best_iter", "<i4"), ("ambiguous", "<i4"), ("replayed", "<i8"),
                          ("priced", "<i4"), ("pad", "<i4")])
REASONS = {2: "boundary", 3: "dependency", 4: "test-failure", 5: "measurement", 6: "hw-safety"}

_u16 = ctypes.POINTER(ctypes.c_uint16)
_u8 = ctypes.POINTER(ctypes.c_uint8)
_i32 = ctypes.POINTER(ctypes.c_int32)


class _Tables(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("words", ctypes.c_int32),
                ("ctrl", ctypes.c_void_p), ("lat", ctypes.c_void_p), ("klass", ctypes.c_void_p),
                ("reads", ctypes.c_void_p), ("writes", ctypes.c_void_p), ("refs", ctypes.c_void_p),
                ("nrefs", ctypes.c_void_p), ("cut", ctypes.c_void_p), ("pin", ctypes.c_void_p),
                ("guard", ctypes.c_void_p)]  # sm100 hardware model: unused by the oracle


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
        L = ctypes.CDLL(str(LIB))
        L.oracle_anneal.argtypes = [ctypes.POINTER(_Tables), ctypes.POINTER(ctypes.c_double),
                                    ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p,
                                    _u16, _u16, ctypes.c_void_p]
        L.oracle_anneal.restype = ctypes.c_int
        L.oracle_simulate_tables.argtypes = [ctypes.POINTER(_Tables), _u16]
        L.oracle_simulate_tables.restype = ctypes.c_int64
        L.oracle_swap_legal.argtypes = [ctypes.POINTER(_Tables), _u16, _u8]
        L.oracle_swap_legal.restype = ctypes.c_long
        L.oracle_sample_inputs.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, _i32, _i32,
                                           _i32, _u8]
        L.oracle_sample_inputs.restype = ctypes.c_int
        _lib = L
    return _lib


class OracleListing:
    """Oracle view over product-independent numpy tables (tables.KernelTables fields)."""

    def __init__(self, t):
        self.t = t
        self.n = t.n
        self._c = _Tables(t.n, t.words, t.ctrl.ctypes.data, t.lat.ctypes.data, t.klass.ctypes.data,
                          t.reads.ctypes.data, t.writes.ctypes.data, t.refs.ctypes.data,
                          t.nrefs.ctypes.data, t.cut.ctypes.data, t.pin.ctypes.data)

    def simulate(self, order) -> int:
        o = np.ascontiguousarray(order, dtype=np.uint16)
        return int(lib().oracle_simulate_tables(ctypes.byref(self._c), o.ctypes.data_as(_u16)))

    def swap_legal(self, order) -> np.ndarray:
        o = np.ascontiguousarray(order, dtype=np.uint16)
        out = np.zeros(max(self.n - 1, 1), dtype=np.uint8)
        lib().oracle_swap_legal(ctypes.byref(self._c), o.ctypes.data_as(_u16), out.ctypes.data_as(_u8))
        return out[: self.n - 1]

    def anneal(self, seed: int, temps, unsafe: bool = False):
        temps = np.ascontiguousarray(temps, dtype=np.float64)
        hist = np.zeros(max(len(temps), 1), dtype=RECORD_DTYPE)
        best = np.zeros(self.n, dtype=np.uint16)
        cur = np.zeros(self.n, dtype=np.uint16)
        summ = np.zeros(1, dtype=SUMMARY_DTYPE)
        rc = lib().oracle_anneal(ctypes.byref(self._c),
                                 temps.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(temps),
                                 int(unsafe), int(seed), hist.ctypes.data, best.ctypes.data_as(_u16),
                                 cur.ctypes.data_as(_u16), summ.ctypes.data)
        if rc != 0:
            raise RuntimeError(f"oracle_anneal failed: {rc}")
        return hist[: len(temps)], best, cur, summ[0]


def history_jsonl(records, t0: float, temps) -> str:
    """Reference HistoryRecord.to_json (anneal.py:87-99) over compact records."""
    lines = []
    t_prev = t0
    for it, r in enumerate(records):
        st = int(r["status"])
        d = {"iteration": it,
             "action": {"candidate": int(r["candidate"]),
                        "direction": "down" if int(r["direction"]) else "up"},
             "temperature": float(temps[it])}
        if st <= 1:
            t = float(r["time"])
            d.update(energy=t / t0, feedback=(t_prev - t) / t0, accepted=st == 0, rejected=None)
            if st == 0:
                t_prev = t
        else:
            d.update(energy=None, feedback=0.0, accepted=False, rejected=REASONS[st])
        lines.append(json.dumps(d, sort_keys=True) + "\n")
    return "".join(lines)


def temperatures(t_max: float, cooling: float, budget: int) -> list:
    out, t = [], t_max
    for _ in range(budget):
        out.append(t)
        t /= cooling
    return out


def sample_inputs(seed: int, index: int, specs) -> list:
    """specs: [(length, cell_bytes, dist_code)] -> list of bytes per buffer."""
    length = np.array([s[0] for s in specs], dtype=np.int32)
    cell = np.array([s[1] for s in specs], dtype=np.int32)
    dist = np.array([s[2] for s in specs], dtype=np.int32)
    total = int((length * cell).sum())
    out = np.zeros(max(total, 1), dtype=np.uint8)
    lib().oracle_sample_inputs(seed, index, len(specs), length.ctypes.data_as(_i32),
                               cell.ctypes.data_as(_i32), dist.ctypes.data_as(_i32),
                               out.ctypes.data_as(_u8))
    res, off = [], 0
    for ln, c, _ in specs:
        res.append(out[off: off + ln * c].tobytes())
        off += ln * c
    return res
