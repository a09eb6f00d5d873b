"""Compiler from SASS listings to the GPU interpreter's ops (csrc/interp.cu).

The supported subset and the compile-time refusals follow the reference's
closure compiler (machine.py:407-654): integer ALU (MOV, IMAD[.WIDE], IADD3,
LEA, LOP3, SHF, SEL, ISETP, IMNMX, IABS, POPC, LDC, S2R...), LDG/LDS/STG/STS/
LDGSTS, guard predicates, EXIT; anything else raises
``UnsupportedInstruction`` at compile time exactly where the reference does.
Constant-bank operands are resolved here from the deterministic buffer layout
(machine.py:29-31, 657-696).  Execution is on the device: ``CompiledKernel.run``
executes one binding; ``difftest`` runs whole sample batches.
"""
from __future__ import annotations

import ctypes
import re
from typing import Mapping

import numpy as np

from .ir import InstrClass, Kernel, Operand, OperandKind

M32 = 0xFFFFFFFF
BUFFER_BASE = 0x10000
BUFFER_ALIGN = 256
PARAM_BANK_BASE = 0x160
SHARED_SIZE = 64 * 1024

OP = {name: i for i, name in enumerate(
    "NOP EXIT MOV ZERO LDC2 IMAD IMADW IADD3 LEA LOP3 SHF SEL ISETP IMNMX IABS POPC LOAD STORE LDGSTS".split())}
SK_IMM, SK_REG, SK_ZERO, SK_UNINIT = 0, 1, 2, 3
MOD = {"": 0, "-": 1, "~": 2, "|": 3}
CMP = {"EQ": 0, "NE": 1, "LT": 2, "LE": 3, "GT": 4, "GE": 5}
COMB = {"AND": 0, "OR": 1, "XOR": 2}
VM_DTYPE = np.dtype([("w", "<i4", 16)])
_REG = re.compile(r"^(U?)R(\d+|Z)$")
_PRED = re.compile(r"^(U?)P(\d+|T)$")


class UnsupportedInstruction(Exception):
    """Instruction outside the interpretable subset."""


class OutOfBoundsAccess(Exception):
    pass


class UninitializedRead(Exception):
    pass


def reg_index(name: str) -> int:
    m = _REG.match(name or "RZ")
    if m is None:
        raise UnsupportedInstruction(f"register {name!r}")
    uni, num = m.group(1), m.group(2)
    if num == "Z":
        return 401 if uni else 300
    k = int(num)
    if (uni and k > 99) or (not uni and k > 299):
        raise UnsupportedInstruction(f"register {name!r} out of range")
    return 301 + k if uni else k


def pred_index(name: str) -> int:
    m = _PRED.match(name or "PT")
    if m is None:
        raise UnsupportedInstruction(f"predicate {name!r}")
    uni, num = m.group(1), m.group(2)
    if num == "T":
        return 17 if uni else 8
    k = int(num)
    if k > 7:
        raise UnsupportedInstruction(f"predicate {name!r} out of range")
    return 9 + k if uni else k


def buffer_bases(lengths: Mapping[int, int]) -> dict:
    """Deterministic guard-separated bases per argument (reference machine.py:657-665)."""
    bases, base = {}, BUFFER_BASE
    for arg in sorted(lengths):
        bases[arg] = base
        span = max(lengths[arg], 1)
        base += (span + BUFFER_ALIGN - 1) // BUFFER_ALIGN * BUFFER_ALIGN + BUFFER_ALIGN
    return bases


def cbank_table(bases: Mapping[int, int]) -> dict:
    cb = {}
    for arg, addr in bases.items():
        slot = PARAM_BANK_BASE + 8 * arg
        cb[slot] = addr & M32
        cb[slot + 4] = (addr >> 32) & M32
    return cb


def _size(ins) -> int:
    for mod in ins.modifiers:
        if mod == "128":
            return 16
        if mod == "64":
            return 8
        if mod in ("U16", "S16", "16"):
            return 2
        if mod in ("U8", "S8", "8"):
            return 1
    return 4


class _Compiler:
    def __init__(self, cbank: Mapping[int, int], strict: bool):
        self.cbank = cbank
        self.strict = strict

    def const(self, bank: int, addr: int):
        if bank != 0:
            return (SK_UNINIT, 0) if self.strict else (SK_IMM, 0)
        v = self.cbank.get(addr)
        if v is None:
            return (SK_UNINIT, 0) if self.strict else (SK_IMM, 0)
        return (SK_IMM, v & M32)

    def src(self, op: Operand, ins) -> tuple:
        if op.kind is OperandKind.IMMEDIATE:
            if not isinstance(op.value, int):
                raise UnsupportedInstruction(f"{ins.mnemonic}: non-integer immediate {op.text}")
            return (SK_IMM, op.value & M32)
        if op.kind in (OperandKind.REGISTER, OperandKind.UREGISTER):
            return (SK_REG | (MOD.get(op.modifier, 0) << 4), reg_index(op.reg or "RZ"))
        if op.kind is OperandKind.CONSTANT:
            return self.const(op.bank or 0, op.addr or 0)
        if op.kind is OperandKind.SPECIAL:
            return (SK_ZERO, 0)
        raise UnsupportedInstruction(f"{ins.mnemonic}: unsupported operand {op.text!r}")

    @staticmethod
    def addr(op: Operand, ins) -> tuple:
        if op.aux_regs:
            raise UnsupportedInstruction(f"{ins.mnemonic}: composite address {op.text!r}")
        base = -1 if op.reg is None else reg_index(op.reg)
        off = op.offset & 0xFFFFFFFFFFFFFFFF
        return base, int(op.base_pair and op.reg is not None), off & M32, (off >> 32) & M32

    @staticmethod
    def dest(ins, slot: int = 0) -> int:
        op = ins.operands[slot]
        if op.kind not in (OperandKind.REGISTER, OperandKind.UREGISTER):
            raise UnsupportedInstruction(f"{ins.mnemonic}: destination must be a register")
        return reg_index(op.reg or "RZ")

    def compile(self, ins) -> list | None:
        """One op (16 words) or None for a no-op; raises UnsupportedInstruction."""
        klass, base = ins.klass, ins.base_mnemonic
        if base == "NOP":
            return None
        if base == "EXIT":
            w = self.new(OP["EXIT"])
        elif klass is InstrClass.BARRIER:
            return None
        elif klass is InstrClass.CONTROL_FLOW:
            raise UnsupportedInstruction(f"{ins.mnemonic}: control flow")
        elif klass is InstrClass.GLOBAL_ASYNC_COPY:
            w = self.ldgsts(ins)
        elif klass in (InstrClass.GLOBAL_LOAD, InstrClass.SHARED_LOAD):
            w = self.load(ins, 1 if klass is InstrClass.SHARED_LOAD else 0)
        elif klass in (InstrClass.GLOBAL_STORE, InstrClass.SHARED_STORE):
            if base in ("RED", "ATOM", "ATOMG", "ATOMS"):
                raise UnsupportedInstruction(ins.mnemonic)
            w = self.store(ins, 1 if klass is InstrClass.SHARED_STORE else 0)
        elif klass is InstrClass.COMPUTE:
            w = self.alu(ins)
        else:
            raise UnsupportedInstruction(ins.mnemonic)
        if ins.predicate and ins.predicate not in ("PT", "UPT"):
            w[1] = pred_index(ins.predicate) | (int(ins.predicate_negated) << 8) | (1 << 9)
        elif ins.predicate and ins.predicate_negated:
            return None  # @!PT never executes
        return w

    @staticmethod
    def new(code: int) -> list:
        w = [0] * 16
        w[0] = code
        return w

    def put(self, w, slot, s):
        w[slot], w[slot + 1] = s[0], s[1]

    def load(self, ins, space):
        ops = ins.operands
        if len(ops) != 2 or ops[0].kind not in (OperandKind.REGISTER, OperandKind.UREGISTER):
            raise UnsupportedInstruction(f"{ins.mnemonic}: unsupported load shape")
        w = self.new(OP["LOAD"])
        w[2] = reg_index(ops[0].reg or "RZ")
        b, pair, lo, hi = self.addr(ops[1], ins)
        w[9], w[10], w[11], w[12], w[13] = space, b, pair, lo, hi
        w[14] = _size(ins)
        w[15] = int(any(m in ("S8", "S16") for m in ins.modifiers))
        return w

    def store(self, ins, space):
        ops = ins.operands
        if len(ops) != 2 or ops[0].kind is not OperandKind.MEMORY:
            raise UnsupportedInstruction(f"{ins.mnemonic}: unsupported store shape")
        if ops[1].kind not in (OperandKind.REGISTER, OperandKind.UREGISTER):
            raise UnsupportedInstruction(f"{ins.mnemonic}: store data must be a register")
        b, pair, lo, hi = self.addr(ops[0], ins)
        w = self.new(OP["STORE"])
        w[2] = reg_index(ops[1].reg or "RZ")
        w[9], w[10], w[11], w[12], w[13] = space, b, pair, lo, hi
        w[14] = _size(ins)
        return w

    def ldgsts(self, ins):
        mem = [op for op in ins.operands if op.kind is OperandKind.MEMORY]
        if len(mem) != 2 or len(ins.operands) != 2:
            raise UnsupportedInstruction(f"{ins.mnemonic}: only plain two-address copies execute")
        w = self.new(OP["LDGSTS"])
        w[2], w[3], w[4], w[5] = self.addr(mem[0], ins)
        w[10], w[11], w[12], w[13] = self.addr(mem[1], ins)
        w[14] = _size(ins)
        return w

    def alu(self, ins):
        base = ins.base_mnemonic
        mods = set(ins.modifiers)
        ops = ins.operands
        if base in ("MOV", "MOV32I", "UMOV"):
            if len(ops) == 3 and not (ops[2].kind is OperandKind.IMMEDIATE and ops[2].value == 0xF):
                raise UnsupportedInstruction(f"{ins.mnemonic}: partial lane mask")
            if len(ops) not in (2, 3):
                raise UnsupportedInstruction(f"{ins.mnemonic}: operand count")
            w = self.new(OP["MOV"])
            w[2] = self.dest(ins)
            self.put(w, 3, self.src(ops[1], ins))
            return w
        if base in ("S2R", "S2UR", "CS2R"):
            w = self.new(OP["ZERO"])
            w[2] = self.dest(ins)
            return w
        if base in ("LDC", "ULDC"):
            if len(ops) != 2 or ops[1].kind is not OperandKind.CONSTANT:
                raise UnsupportedInstruction(f"{ins.mnemonic}: shape")
            w = self.new(OP["LDC2"])
            w[2] = self.dest(ins)
            self.put(w, 3, self.const(ops[1].bank or 0, ops[1].addr or 0))
            self.put(w, 5, self.const(ops[1].bank or 0, (ops[1].addr or 0) + 4))
            w[9] = 2 if "64" in mods else 1
            nxt = ops[0].reg or "RZ"
            m = re.match(r"^(U?R)(\d+)$", nxt)
            w[10] = reg_index(f"{m.group(1)}{int(m.group(2)) + 1}") if m else reg_index(nxt)
            return w
        if base in ("IMAD", "UIMAD"):
            if any(m in mods for m in ("HI", "X")):
                raise UnsupportedInstruction(f"{ins.mnemonic}: carry/high forms")
            if len(ops) != 4:
                raise UnsupportedInstruction(f"{ins.mnemonic}: operand count")
            if "WIDE" in mods:
                w = self.new(OP["IMADW"])
                w[2] = self.dest(ins)
                self.put(w, 3, self.src(ops[1], ins))
                self.put(w, 5, self.src(ops[2], ins))
                w[9] = int("U32" in mods)
                acc = ops[3]
                if acc.kind in (OperandKind.REGISTER, OperandKind.UREGISTER):
                    if acc.modifier:
                        raise UnsupportedInstruction(f"{ins.mnemonic}: modified accumulator")
                    w[10], w[11] = 0, reg_index(acc.reg or "RZ")
                elif acc.kind is OperandKind.IMMEDIATE and isinstance(acc.value, int):
                    v = acc.value & 0xFFFFFFFFFFFFFFFF
                    w[10], w[11], w[12] = 1, v & M32, v >> 32
                else:
                    raise UnsupportedInstruction(f"{ins.mnemonic}: accumulator {acc.text!r}")
                return w
            w = self.new(OP["IMAD"])
            w[2] = self.dest(ins)
            for k, slot in ((1, 3), (2, 5), (3, 7)):
                self.put(w, slot, self.src(ops[k], ins))
            return w
        if base in ("IADD3", "UIADD3"):
            if len(ops) != 4 or any(op.kind is OperandKind.PREDICATE for op in ops):
                raise UnsupportedInstruction(f"{ins.mnemonic}: carry-predicate form")
            w = self.new(OP["IADD3"])
            w[2] = self.dest(ins)
            for k, slot in ((1, 3), (2, 5), (3, 7)):
                self.put(w, slot, self.src(ops[k], ins))
            return w
        if base in ("LEA", "ULEA"):
            if mods - {"U32"}:
                raise UnsupportedInstruction(f"{ins.mnemonic}: mods {sorted(mods)}")
            if len(ops) == 3:
                shift = 0
            elif len(ops) == 4 and ops[3].kind is OperandKind.IMMEDIATE and isinstance(ops[3].value, int):
                shift = ops[3].value & 31
            else:
                raise UnsupportedInstruction(f"{ins.mnemonic}: shape")
            w = self.new(OP["LEA"])
            w[2] = self.dest(ins)
            self.put(w, 3, self.src(ops[1], ins))
            self.put(w, 5, self.src(ops[2], ins))
            w[9] = shift
            return w
        if base in ("LOP3", "ULOP3"):
            if "LUT" not in mods or len(ops) < 5:
                raise UnsupportedInstruction(f"{ins.mnemonic}: shape")
            if len(ops) == 6:
                tail = ops[5]
                if not (tail.kind is OperandKind.PREDICATE and tail.reg in ("PT", "UPT")):
                    raise UnsupportedInstruction(f"{ins.mnemonic}: predicate output")
            elif len(ops) != 5:
                raise UnsupportedInstruction(f"{ins.mnemonic}: operand count")
            if not (ops[4].kind is OperandKind.IMMEDIATE and isinstance(ops[4].value, int)):
                raise UnsupportedInstruction(f"{ins.mnemonic}: LUT immediate")
            w = self.new(OP["LOP3"])
            w[2] = self.dest(ins)
            for k, slot in ((1, 3), (2, 5), (3, 7)):
                self.put(w, slot, self.src(ops[k], ins))
            w[9] = ops[4].value & 0xFF
            return w
        if base in ("SHF", "USHF"):
            left, right = "L" in mods, "R" in mods
            if left == right or not mods & {"U32", "S32"}:
                raise UnsupportedInstruction(f"{ins.mnemonic}: form")
            if len(ops) != 4:
                raise UnsupportedInstruction(f"{ins.mnemonic}: operand count")
            w = self.new(OP["SHF"])
            w[2] = self.dest(ins)
            for k, slot in ((1, 3), (2, 5), (3, 7)):
                self.put(w, slot, self.src(ops[k], ins))
            w[9] = int(left) | (int("S32" in mods) << 1) | (int("HI" in mods) << 2)
            return w
        if base in ("SEL", "USEL"):
            if len(ops) != 4 or ops[3].kind is not OperandKind.PREDICATE:
                raise UnsupportedInstruction(f"{ins.mnemonic}: shape")
            w = self.new(OP["SEL"])
            w[2] = self.dest(ins)
            self.put(w, 3, self.src(ops[1], ins))
            self.put(w, 5, self.src(ops[2], ins))
            w[9], w[10] = pred_index(ops[3].reg or "PT"), int(ops[3].modifier == "!")
            return w
        if base in ("ISETP", "UISETP"):
            cmp_name = next((m for m in ins.modifiers if m in CMP), None)
            comb_name = next((m for m in ins.modifiers if m in COMB), None)
            if cmp_name is None or comb_name is None or "EX" in mods:
                raise UnsupportedInstruction(f"{ins.mnemonic}: form")
            if len(ops) != 5 or ops[0].kind is not OperandKind.PREDICATE:
                raise UnsupportedInstruction(f"{ins.mnemonic}: shape")
            if not (ops[1].kind is OperandKind.PREDICATE and ops[1].reg in ("PT", "UPT")):
                raise UnsupportedInstruction(f"{ins.mnemonic}: dual predicate outputs")
            w = self.new(OP["ISETP"])
            w[2] = pred_index(ops[0].reg or "PT")
            self.put(w, 3, self.src(ops[2], ins))
            self.put(w, 5, self.src(ops[3], ins))
            w[9], w[10], w[11] = CMP[cmp_name], COMB[comb_name], int("U32" in mods)
            w[12], w[13] = pred_index(ops[4].reg or "PT"), int(ops[4].modifier == "!")
            return w
        if base == "IMNMX":
            if len(ops) != 4 or ops[3].kind is not OperandKind.PREDICATE:
                raise UnsupportedInstruction(f"{ins.mnemonic}: shape")
            w = self.new(OP["IMNMX"])
            w[2] = self.dest(ins)
            self.put(w, 3, self.src(ops[1], ins))
            self.put(w, 5, self.src(ops[2], ins))
            w[9], w[10] = pred_index(ops[3].reg or "PT"), int(ops[3].modifier == "!")
            w[11] = int("U32" in mods)
            return w
        if base == "IABS" or base in ("POPC", "UPOPC"):
            if len(ops) != 2:
                raise UnsupportedInstruction(f"{ins.mnemonic}: shape")
            w = self.new(OP["IABS" if base == "IABS" else "POPC"])
            w[2] = self.dest(ins)
            self.put(w, 3, self.src(ops[1], ins))
            return w
        raise UnsupportedInstruction(ins.mnemonic)


def compile_kernel(kernel: Kernel, lengths: Mapping[int, int], *, strict: bool = False) -> np.ndarray:
    """Ops for the device VM (raises UnsupportedInstruction)."""
    comp = _Compiler(cbank_table(buffer_bases(lengths)), strict)
    prog = [w for w in (comp.compile(ins) for ins in kernel.schedule) if w is not None]
    arr = np.zeros(len(prog), dtype=VM_DTYPE)
    for i, w in enumerate(prog):
        arr[i]["w"] = [int(x) - (1 << 32) if int(x) >= (1 << 31) else int(x) for x in w]
    return arr


def touches_shared(kernel: Kernel) -> bool:
    return any(ins.klass in (InstrClass.SHARED_LOAD, InstrClass.SHARED_STORE, InstrClass.GLOBAL_ASYNC_COPY)
               for ins in kernel.schedule)


class CompiledKernel:
    """Kernel checked against the interpretable subset (reference machine.py:668-711).

    Construction validates every instruction (``UnsupportedInstruction``);
    ``run`` executes one input binding on the device.
    """

    def __init__(self, kernel: Kernel, *, strict: bool = False, shared_size: int = SHARED_SIZE):
        self.kernel = kernel
        self.strict = strict
        self.shared_size = shared_size if touches_shared(kernel) else 0
        comp = _Compiler({}, strict)
        for ins in kernel.schedule:  # validate once; constants are bound per layout in program()
            comp.compile(ins)
        self._progs: dict = {}

    def program(self, lengths: Mapping[int, int]) -> np.ndarray:
        key = tuple(sorted(lengths.items()))
        if key not in self._progs:
            self._progs[key] = compile_kernel(self.kernel, dict(key), strict=self.strict)
        return self._progs[key]

    def run(self, buffers: Mapping[int, bytes], ret_ptr: int) -> bytes:
        if ret_ptr not in buffers:
            raise ValueError(f"ret_ptr {ret_ptr} is not a bound buffer")
        from .vm import run_bindings

        outs, status, fault = run_bindings(self, [dict(buffers)])
        if status[0] == 1:
            raise OutOfBoundsAccess(f"global access at {fault[0]:#x}")
        if status[0] == 2:
            raise OutOfBoundsAccess(f"shared access at {fault[0]:#x}")
        if status[0] == 3:
            raise UninitializedRead(f"register id {fault[0]}")
        return outs[0][ret_ptr]


def interpret(kernel: Kernel, buffers: Mapping[int, bytes], ret_ptr: int, *, strict: bool = False) -> bytes:
    return CompiledKernel(kernel, strict=strict).run(buffers, ret_ptr)
