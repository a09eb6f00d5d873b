"""Cubin frontend (G3): sm_100a kernel -> reference text listing -> permuted cubin.

* Words, pins and patching come from libsip (``sip_module_*``, C++ ELF code).
* Mnemonics/operands and branch-target labels come from ``nvdisasm -c -hex``
  (cuobjdump prints no labels, so branch targets would not become cuts --
  SURVEY appendix A2).
* Control codes are decoded from bits 105..127 of each instruction
  (hi64 >> 41): stall [3:0], yield [4] ('Y' printed when the bit is 0),
  write barrier [7:5], read barrier [10:8], wait mask [16:11], reuse [20:17].
* Each instruction renders on ONE line in the reference's format with both
  64-bit words in a trailing comment, e.g.
  ``        /*0670*/ [B------:R0:W-:Y:S12] @!UP1 UTCHMMA ... ; /* 0x... 0x... */``
  The address comment is the instruction's identity: a permuted schedule maps
  back to a word permutation by reading it.
"""
from __future__ import annotations

import ctypes
import re
import shutil
import subprocess
import tempfile
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .engine import c_u8p, c_u16p, c_u64p, load_library
from .ir import Kernel
from .sasstext import parse_kernel

_ADDR = re.compile(r"^\s*/\*([0-9a-f]{4,})\*/\s*(.*?)\s*;\s*/\*\s*(0x[0-9a-f]{16})\s*\*/\s*$")
_HI = re.compile(r"^\s*/\*\s*(0x[0-9a-f]{16})\s*\*/\s*$")
_LABEL = re.compile(r"^\s*(\.L_x_\d+|[A-Za-z_.$][\w.$]*):\s*$")
_ADDR_ID = re.compile(r"/\*([0-9a-f]{4,})\*/")


def decode_control(hi: int) -> tuple:
    """(text, reuse) for the 64-bit high word of one sm_100a instruction."""
    c = (hi >> 41) & 0x7FFFFF
    stall = c & 0xF
    yld = "Y" if not (c >> 4) & 1 else "-"
    wr = (c >> 5) & 7
    rd = (c >> 8) & 7
    wait = (c >> 11) & 0x3F
    reuse = (c >> 17) & 0xF
    slots = "".join(str(b) if (wait >> b) & 1 else "-" for b in range(6))
    rds = "-" if rd == 7 else str(rd)
    wrs = "-" if wr == 7 else str(wr)
    return f"[B{slots}:R{rds}:W{wrs}:{yld}:S{stall:02d}]", reuse


class Module:
    """A cubin opened through libsip (parse-only when ctx is None)."""

    def __init__(self, cubin: bytes, func: str, ctx=None):
        self.lib = load_library()
        self.ctx = ctx
        self.cubin = bytes(cubin)
        self.func = func
        self._buf = ctypes.create_string_buffer(self.cubin, len(self.cubin))
        h = ctypes.c_void_p()
        rc = self.lib.sip_module_open(ctx.handle if ctx else None, self._buf, len(self.cubin),
                                      func.encode(), ctypes.byref(h))
        if rc != 0:
            msg = ctx.lib.sip_last_error(ctx.handle).decode() if ctx else f"code {rc}"
            raise ValueError(f"cannot open {func} in cubin: {msg}")
        self.handle = h
        n = ctypes.c_int32()
        off = ctypes.c_uint64()
        self.lib.sip_module_info(h, ctypes.byref(n), ctypes.byref(off))
        self.n = n.value
        self.text_offset = off.value

    def words(self) -> np.ndarray:
        w = np.zeros(2 * self.n, dtype=np.uint64)
        self.lib.sip_module_words(self.handle, w.ctypes.data_as(c_u64p))
        return w.reshape(self.n, 2)

    def pins(self) -> np.ndarray:
        p = np.zeros(self.n, dtype=np.uint8)
        self.lib.sip_module_pins(self.handle, p.ctypes.data_as(c_u8p))
        return p

    def patch(self, perm) -> bytes:
        perm = np.ascontiguousarray(perm, dtype=np.uint16)
        size = ctypes.c_size_t(0)
        self.lib.sip_module_patch(self.handle, perm.ctypes.data_as(c_u16p), None, ctypes.byref(size))
        out = ctypes.create_string_buffer(size.value)
        rc = self.lib.sip_module_patch(self.handle, perm.ctypes.data_as(c_u16p), out, ctypes.byref(size))
        if rc != 0:
            raise ValueError(f"patch failed ({rc})")
        return out.raw[: size.value]

    def close(self) -> None:
        if self.handle:
            self.lib.sip_module_close(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nvdisasm_text(cubin: bytes) -> str:
    exe = shutil.which("nvdisasm") or "/usr/local/cuda/bin/nvdisasm"
    with tempfile.NamedTemporaryFile(suffix=".cubin") as fh:
        fh.write(cubin)
        fh.flush()
        res = subprocess.run([exe, "-c", "-hex", fh.name], capture_output=True, text=True, check=True)
    return res.stdout


@dataclass
class Listing:
    func: str
    text: str
    kernel: Kernel
    words: np.ndarray      # [n, 2] uint64, identity order
    pins: np.ndarray       # [n] uint8
    reuse: list            # [n] reuse bits per identity

    @property
    def n(self) -> int:
        return len(self.kernel.schedule)


def render_listing(cubin: bytes, func: str) -> Listing:
    """Decode one kernel of a cubin into the reference text format."""
    mod = Module(cubin, func)
    words = mod.words()
    pins = mod.pins()
    mod.close()
    dis = nvdisasm_text(cubin).splitlines()
    sect = f".text.{func}"
    out, reuse = [], []
    inside = False
    i = 0
    while i < len(dis):
        line = dis[i]
        if line.strip().startswith(".section"):
            inside = sect in line.split(",")[0].split()
            if inside:
                out.append(f"\t.section\t{sect}")
            i += 1
            continue
        if not inside:
            i += 1
            continue
        m = _ADDR.match(line)
        if m:
            addr = int(m.group(1), 16)
            lo = int(m.group(3), 16)
            hm = _HI.match(dis[i + 1]) if i + 1 < len(dis) else None
            if hm is None:
                raise ValueError(f"instruction at {addr:#x} lacks its second word")
            hi = int(hm.group(1), 16)
            idx = addr // 16
            if idx >= len(words) or int(words[idx, 0]) != lo or int(words[idx, 1]) != hi:
                raise ValueError(f"nvdisasm word mismatch at {addr:#x}")
            ctrl, ru = decode_control(hi)
            body = " ".join(m.group(2).split())
            out.append(f"        /*{addr:04x}*/ {ctrl} {body} ; /* {lo:#018x} {hi:#018x} */")
            reuse.append(ru)
            i += 2
            continue
        lm = _LABEL.match(line)
        if lm:
            out.append(f"{lm.group(1)}:")
        elif line.strip().startswith("."):
            out.append("\t" + line.strip())
        i += 1
    text = "\n".join(out) + "\n"
    kernel = parse_kernel(text, name=func)
    if len(kernel.schedule) != len(words):
        raise ValueError(f"listing has {len(kernel.schedule)} instructions, .text has {len(words)}")
    for k, ins in enumerate(kernel.schedule):
        if identity_of(ins) != k:
            raise ValueError(f"instruction {k} out of order in the listing")
    return Listing(func, text, kernel, words, pins, reuse)


def identity_of(ins) -> int:
    """Original slot of an instruction rendered by render_listing (its /*addr*/ comment)."""
    m = _ADDR_ID.search(ins.source_text or "")
    if m is None:
        raise ValueError("instruction carries no address comment")
    return int(m.group(1), 16) // 16


def schedule_perm(kernel: Kernel) -> np.ndarray:
    """Word permutation realising a (permuted) listing schedule."""
    return np.array([identity_of(ins) for ins in kernel.schedule], dtype=np.uint16)


def load_cubin(path) -> bytes:
    return Path(path).read_bytes()
