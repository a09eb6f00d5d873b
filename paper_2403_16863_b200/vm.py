"""Device orchestration of the interpreter: sample batches in HBM, two programs, compare.

Per batch of samples: the reference's sample stream is generated straight
into a device region ``[count][stride]`` (``sip_sample_inputs_device``), the
region is duplicated, the reference program runs on one copy and the mutant on
the other (``sip_vm_exec``, one thread per sample), and the ret buffers are
compared cell by cell (``sip_vm_cell_diff``).  Only per-sample outcome codes
come back to the host.  torch is used for device allocation only.
"""
from __future__ import annotations

import ctypes

import numpy as np

from .engine import c_i32p, c_i64p, get_context
from .interp import buffer_bases

CELL = {"int8": 1, "int16": 2, "int32": 4}
DIST = {"uniform": 0, "small": 1, "zero": 2}


class Layout:
    """Where each plan buffer lives: virtual base, length, offset inside a sample slice."""

    def __init__(self, specs):
        self.args = [s.arg for s in specs]
        self.nbytes = np.array([s.nbytes for s in specs], dtype=np.int32)
        self.cell = np.array([CELL[s.kind] for s in specs], dtype=np.int32)
        self.dist = np.array([DIST[s.dist] for s in specs], dtype=np.int32)
        self.offs = np.concatenate([[0], np.cumsum(self.nbytes)[:-1]]).astype(np.int32)
        self.stride = int(self.nbytes.sum())
        bases = buffer_bases({s.arg: s.nbytes for s in specs})
        self.bases = np.array([bases[a] for a in self.args], dtype=np.int64)
        self.lengths = {s.arg: s.nbytes for s in specs}

    def offset_of(self, arg) -> int:
        return int(self.offs[self.args.index(arg)])


def _torch():
    import torch

    return torch


def exec_program(ctx, ck, layout: Layout, region, count: int):
    prog = ck.program(layout.lengths)
    status = np.zeros(count, dtype=np.int32)
    fault = np.zeros(count, dtype=np.int64)
    ctx.check(ctx.lib.sip_vm_exec(ctx.handle, prog.ctypes.data_as(ctypes.c_void_p), len(prog), len(layout.args),
                                  layout.bases.ctypes.data_as(c_i64p), layout.nbytes.ctypes.data_as(c_i32p),
                                  layout.offs.ctypes.data_as(c_i32p), ctypes.c_void_p(region.data_ptr()),
                                  layout.stride, count, ck.shared_size, int(ck.strict),
                                  status.ctypes.data_as(c_i32p), fault.ctypes.data_as(c_i64p)))
    return status, fault


def run_batch(ref_ck, mut_ck, plan, first: int, count: int, ret_ptr: int):
    """Run both programs on samples [first, first+count) of the plan's stream."""
    torch = _torch()
    ctx = get_context()
    layout = Layout(plan.buffers)
    a = torch.empty(count * max(layout.stride, 1), dtype=torch.uint8, device="cuda")
    ctx.check(ctx.lib.sip_sample_inputs_device(ctx.handle, plan.seed, first, count, len(layout.args),
                                               layout.nbytes.ctypes.data_as(c_i32p),
                                               layout.cell.ctypes.data_as(c_i32p),
                                               layout.dist.ctypes.data_as(c_i32p),
                                               ctypes.c_void_p(a.data_ptr())))
    b = a.clone()
    st_ref, f_ref = exec_program(ctx, ref_ck, layout, a, count)
    st_mut, f_mut = exec_program(ctx, mut_ck, layout, b, count)
    off = layout.offset_of(ret_ptr)
    k = layout.args.index(ret_ptr)
    cells = np.zeros(count, dtype=np.int32)
    ctx.check(ctx.lib.sip_vm_cell_diff(ctx.handle, ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
                                       layout.stride, off, int(layout.nbytes[k]), int(layout.cell[k]), count,
                                       cells.ctypes.data_as(c_i32p)))
    return {"layout": layout, "a": a, "b": b, "st_ref": st_ref, "f_ref": f_ref, "st_mut": st_mut,
            "f_mut": f_mut, "cells": cells}


def run_bindings(ck, bindings: list):
    """Execute explicit host bindings (dict arg -> bytes) on the device; returns outputs."""
    torch = _torch()
    ctx = get_context()
    args = sorted(bindings[0])
    lengths = {a: len(bindings[0][a]) for a in args}
    offs = np.concatenate([[0], np.cumsum([lengths[a] for a in args])[:-1]]).astype(np.int32)
    stride = int(sum(lengths.values()))
    host = np.zeros((len(bindings), max(stride, 1)), dtype=np.uint8)
    for i, bd in enumerate(bindings):
        for a, o in zip(args, offs):
            host[i, o: o + lengths[a]] = np.frombuffer(bytes(bd[a]), dtype=np.uint8)
    dev = torch.from_numpy(host.reshape(-1)).cuda()
    bases = buffer_bases(lengths)
    prog = ck.program(lengths)
    n = len(bindings)
    status = np.zeros(n, dtype=np.int32)
    fault = np.zeros(n, dtype=np.int64)
    b_arr = np.array([bases[a] for a in args], dtype=np.int64)
    l_arr = np.array([lengths[a] for a in args], dtype=np.int32)
    ctx.check(ctx.lib.sip_vm_exec(ctx.handle, prog.ctypes.data_as(ctypes.c_void_p), len(prog), len(args),
                                  b_arr.ctypes.data_as(c_i64p), l_arr.ctypes.data_as(c_i32p),
                                  offs.ctypes.data_as(c_i32p), ctypes.c_void_p(dev.data_ptr()), stride, n,
                                  ck.shared_size, int(ck.strict), status.ctypes.data_as(c_i32p),
                                  fault.ctypes.data_as(c_i64p)))
    out = dev.cpu().numpy().reshape(n, -1)
    results = [{a: out[i, o: o + lengths[a]].tobytes() for a, o in zip(args, offs)} for i in range(n)]
    return results, (status & 0xFF).tolist(), fault.tolist()
