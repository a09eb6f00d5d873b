"""Synthetic listings for the acceptance tests (independent re-implementations of
the reference test-suite families: latency hiding, corridors, random straight-line
integer programs with a Python evaluator).  Pure text builders; no package code."""
from __future__ import annotations

import random

M32 = 0xFFFFFFFF


def plain(stall: int) -> str:
    return f"[B------:R-:W-:-:S{stall:02d}]"


def setw(bar: int, stall: int) -> str:
    return f"[B------:R-:W{bar}:-:S{stall:02d}]"


def waits(bars, stall: int) -> str:
    return "[B" + "".join(str(b) if b in bars else "-" for b in range(6)) + f":R-:W-:-:S{stall:02d}]"


def hiding(pads: int, stall: int, load_at: int | None = None) -> str:
    """`pads` independent ALU pads, one global load and its consumer."""
    load_at = pads if load_at is None else load_at
    out = []
    for i in range(pads + 1):
        if i == load_at:
            out.append(f"{setw(0, 1)} LDG.E R4, [R2.64] ;")
        if i < pads:
            out.append(f"{plain(stall)} IADD3 R{20 + i}, RZ, 0x1, RZ ;")
    out.append(f"{waits({0}, 1)} IADD3 R5, R4, 0x1, RZ ;")
    return "\n".join(out) + "\n"


def hiding_cycles(pads_before: int, stall: int, mem: int = 400, alu: int = 4) -> int:
    """Closed form of hiding(): the load issues after the pads ahead of it."""
    return pads_before * stall + mem + alu


def corridor(segments) -> str:
    """Each segment: pad run, load, consumer; the consumer feeds the next segment,
    so every load is confined to its own pad run."""
    out, base = [], "R2"
    for s, (pads, stall) in enumerate(segments):
        tie = f"R{60 + 2 * (s - 1)}" if s else "RZ"
        for i in range(pads):
            out.append(f"{plain(stall)} IADD3 R{100 + 10 * s + i}, {tie}, 0x1, RZ ;")
        bar = s % 6
        out.append(f"{setw(bar, 1)} LDG.E R{4 + s}, [{base}.64] ;")
        out.append(f"{waits({bar}, 1)} IADD3 R{60 + 2 * s}, R{4 + s}, 0x1, RZ ;")
        base = f"R{60 + 2 * s}"
    return "\n".join(out) + "\n"


def program(seed: int, ops: int = 8, inputs: int = 4):
    """Random straight-line integer program: loads `inputs` words of arg 0, applies
    `ops` ALU steps, stores 4 words to arg 1.  Returns (text, evaluate(words))."""
    rng = random.Random(seed)
    lines = [f"{plain(1)} MOV R2, c[0x0][0x160] ;", f"{plain(1)} MOV R3, c[0x0][0x164] ;",
             f"{plain(1)} MOV R8, c[0x0][0x168] ;", f"{plain(1)} MOV R9, c[0x0][0x16c] ;"]
    fns, regs, nxt = [], [], 10
    for i in range(inputs):
        lines.append(f"{setw(i, 1)} LDG.E R{nxt}, [R2.64+{hex(4 * i)}] ;")
        fns.append(lambda x, i=i: x[i])
        regs.append(nxt)
        nxt += 1
    lines.append(f"{waits(set(range(inputs)), 1)} IADD3 R{nxt}, RZ, RZ, RZ ;")
    fns.append(lambda x: 0)
    regs.append(nxt)
    nxt += 1
    for _ in range(ops):
        a, b = rng.randrange(len(fns)), rng.randrange(len(fns))
        fa, fb, ra, rb = fns[a], fns[b], regs[a], regs[b]
        kind = rng.choice(["add", "mad", "and", "or", "xor", "shl", "shr", "popc"])
        rd = nxt
        nxt += 1
        if kind == "add":
            lines.append(f"{plain(2)} IADD3 R{rd}, R{ra}, R{rb}, RZ ;")
            f = lambda x, fa=fa, fb=fb: (fa(x) + fb(x)) & M32
        elif kind == "mad":
            k = rng.randrange(1, 16)
            lines.append(f"{plain(2)} IMAD R{rd}, R{ra}, {hex(k)}, R{rb} ;")
            f = lambda x, fa=fa, fb=fb, k=k: (fa(x) * k + fb(x)) & M32
        elif kind in ("and", "or", "xor"):
            lut = {"and": 0xC0, "or": 0xFC, "xor": 0x3C}[kind]
            lines.append(f"{plain(1)} LOP3.LUT R{rd}, R{ra}, R{rb}, RZ, {hex(lut)}, !PT ;")
            op = {"and": lambda p, q: p & q, "or": lambda p, q: p | q, "xor": lambda p, q: p ^ q}[kind]
            f = lambda x, fa=fa, fb=fb, op=op: op(fa(x), fb(x))
        elif kind == "shl":
            k = rng.randrange(31)
            lines.append(f"{plain(1)} SHF.L.U32 R{rd}, R{ra}, {hex(k)}, RZ ;")
            f = lambda x, fa=fa, k=k: (fa(x) << k) & M32
        elif kind == "shr":
            k = rng.randrange(31)
            lines.append(f"{plain(1)} SHF.R.U32 R{rd}, R{ra}, {hex(k)}, RZ ;")
            f = lambda x, fa=fa, k=k: fa(x) >> k
        else:
            lines.append(f"{plain(2)} POPC R{rd}, R{ra} ;")
            f = lambda x, fa=fa: bin(fa(x)).count("1")
        fns.append(f)
        regs.append(rd)
    outs = [rng.randrange(len(fns)) for _ in range(4)]
    for j, v in enumerate(outs):
        lines.append(f"{plain(2)} STG.E [R8.64+{hex(4 * j)}], R{regs[v]} ;")
    lines.append(f"{plain(5)} EXIT ;")
    return "\n".join(lines) + "\n", (lambda words: [fns[v](words) for v in outs])
