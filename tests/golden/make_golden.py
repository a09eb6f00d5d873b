"""Generate golden fixtures by running the *reference* package in this container.

    python tests/golden/make_golden.py            # writes tests/golden/reference.json.gz

The reference (``/root/reference/pkg/src/sasstune``) is importable here but
does not exist on the GPU box, so its outputs are frozen into a committed,
gzipped JSON fixture.  Every listing's text is stored alongside its results
so the tests never need the reference at run time.

Contents per listing: register read/write sets and memory references per
instruction (deps.reads_writes / deps.mem_refs), block cuts, candidate
positions, the simulate() report, adjacent-swap legality verdicts sampled
along random walks (deps.swap_legal), and full annealing outcomes
(anneal.anneal with SimulatorBackend) for a range of seeds and configs.
Also: difftest.sample_inputs byte streams.
"""
from __future__ import annotations

import gzip
import hashlib
import json
import random
import sys
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REF_TESTS))

import kernels as refk  # noqa: E402  (reference test oracles; text builders only)
import sasstune as ref  # noqa: E402
from sasstune.deps import build_depgraph, mem_refs, reads_writes, swap_legal  # noqa: E402

OUT = Path(__file__).with_name("reference.json.gz")
EXTRA = Path(__file__).with_name("listings")  # decoded sm_100a listings (cubin frontend output)


def synthetic_mix(seed: int, n: int = 160) -> str:
    """Random but parseable listing mixing every class the analysis models."""
    rng = random.Random(seed)
    lines = []
    for i in range(n):
        bars = rng.sample(range(6), rng.choice([0, 0, 0, 1, 2]))
        wait = "".join(str(b) if b in bars else "-" for b in range(6))
        rd = rng.choice(["-"] * 6 + [str(rng.randrange(6))])
        wr = rng.choice(["-"] * 3 + [str(rng.randrange(6))])
        ctrl = f"[B{wait}:R{rd}:W{wr}:{rng.choice('-Y')}:S{rng.randrange(16):02d}]"
        r = lambda: f"R{rng.randrange(2, 40)}"  # noqa: E731
        kind = rng.random()
        if kind < 0.14:
            body = f"LDG.E{rng.choice(['', '.64', '.128', '.U8'])} {r()}, [R{2 * rng.randrange(1, 8)}.64+{hex(16 * rng.randrange(8))}]"
        elif kind < 0.26:
            body = f"STG.E{rng.choice(['', '.64', '.128'])} [R{2 * rng.randrange(1, 8)}.64+{hex(16 * rng.randrange(8))}], {r()}"
        elif kind < 0.32:
            body = f"LDGSTS.E.BYPASS.128 [R{rng.randrange(200, 204)}+{hex(0x800 * rng.randrange(4))}], desc[UR16][R{2 * rng.randrange(5, 9)}.64], P0"
        elif kind < 0.40:
            body = f"LDS {r()}, [R{rng.randrange(2, 6)}+{hex(4 * rng.randrange(8))}]"
        elif kind < 0.46:
            body = f"STS [R{rng.randrange(2, 6)}+{hex(4 * rng.randrange(8))}], {r()}"
        elif kind < 0.48:
            body = rng.choice(["BAR.SYNC.DEFER_BLOCKING 0x0", "LDGDEPBAR", "DEPBAR.LE SB0, 0x1"])
        elif kind < 0.58:
            body = f"IMAD.WIDE {r()}, {r()}, 0x4, R{2 * rng.randrange(1, 8)}"
        elif kind < 0.64:
            body = f"ISETP.GE.AND P{rng.randrange(4)}, PT, {r()}, 0x20, PT"
        elif kind < 0.68:
            body = f"@P{rng.randrange(4)} IADD3 {r()}, {r()}, 0x1, RZ"
        elif kind < 0.70:
            body = f"RED.E.ADD.STRONG.GPU [R{2 * rng.randrange(1, 8)}.64], {r()}"
        elif kind < 0.72:
            body = f"UTMALDG.2D [UR{rng.randrange(4, 12)}], [UR{rng.randrange(12, 16)}]"
        else:
            body = f"{rng.choice(['IADD3', 'LOP3.LUT', 'FFMA', 'IMAD', 'POPC'])} {r()}, {r()}, {r()}, RZ"
        if "@P" in body:
            lines.append(f"{ctrl} {body} ;")
        else:
            lines.append(f"{ctrl} {body} ;")
        if rng.random() < 0.04:
            lines.append(f".L_x_{i}:")
    lines.append("[B------:R-:W-:-:S05] EXIT ;")
    return "\n".join(lines) + "\n"


def corpus() -> dict:
    items = {}
    for p in sorted((REF_TESTS / "data").glob("*.sass")):
        items[p.stem] = p.read_text()
    items["hide"] = refk.hiding_kernel(4, 8)
    items["hide_7_5"] = refk.hiding_kernel(7, 5)
    items["interp_hide"] = refk.interp_hiding_kernel(5, 6, 5)
    items["corridor"] = refk.corridor_kernel([(3, 4), (2, 8), (4, 2), (1, 15)])
    items["base_detect"] = refk.BASE_DETECT
    for s in range(6):
        items[f"random_program_{s}"] = refk.random_program(s, n_ops=14, n_inputs=4)[0]
    for s in range(3):
        items[f"synthetic_mix_{s}"] = synthetic_mix(s)
    if EXTRA.is_dir():
        for p in sorted(EXTRA.glob("*.sass")):
            items[p.stem] = p.read_text()
    return items


def perm_of(kernel, sched) -> list:
    ident = {id(ins): i for i, ins in enumerate(kernel.schedule)}
    return [ident[id(ins)] for ins in sched]


def walk_legality(kernel, seed: int, steps: int, max_queries: int) -> list:
    """(perm, [legal per adjacent slot]) along an unsafe random walk."""
    rng = random.Random(1000 + seed)
    k = kernel
    out = []
    n = len(k.schedule)
    if n < 2:
        return out
    cset = ref.candidates(k)
    for step in range(steps):
        if step % max(1, steps // max_queries) == 0:
            g = build_depgraph(k)
            out.append({"perm": perm_of(kernel, k.schedule),
                        "legal": [int(swap_legal(g, k, p)) for p in range(n - 1)]})
        if not cset.positions:
            break
        g = build_depgraph(k)
        act = ref.sample_action(ref.candidates(k), rng)
        try:
            k = ref.apply_action(k, g, act, unsafe=True)
        except ref.MoveRejected:
            pass
    return out


def anneal_record(kernel, cfg, full: bool) -> dict:
    st = ref.anneal(kernel, ref.SimulatorBackend(), cfg)
    jsonl = st.history_jsonl()
    rec = {
        "sha256": hashlib.sha256(jsonl.encode()).hexdigest(),
        "best": perm_of(kernel, st.best.schedule),
        "current": perm_of(kernel, st.current.schedule),
        "best_energy": st.best_energy,
        "current_energy": st.current_energy,
        "baseline": st.baseline,
        "iterations": st.iterations,
        "priced": sum(1 for r in st.history if r.energy is not None),
    }
    if full:
        rec["jsonl"] = jsonl
    return rec


CONFIGS = {
    "default": {},
    "unsafe": {"unsafe_moves": True},
    "long": {"cooling": 1.01, "t_min": 0.001},
    "hot": {"t_max": 8.0, "t_min": 0.5, "cooling": 1.02},
}


def listing_record(name: str, text: str, n_seeds: int) -> dict:
    k = ref.parse_kernel(text, name=name)
    rw = [reads_writes(ins) for ins in k.schedule]
    rec = {
        "text": text,
        "n": len(k.schedule),
        "rw": [[sorted(r), sorted(w)] for r, w in rw],
        "refs": [[[m.space, m.base, m.offset, m.size, int(m.write)] for m in mem_refs(ins)]
                 for ins in k.schedule],
        "cuts": list(k.block_boundaries),
        "cands": list(ref.candidates(k).positions),
        "classes": [ins.klass.value for ins in k.schedule],
        "serialize_ok": ref.serialize_kernel(k) == ref.sasstext.normalize_newlines(text),
        "walks": walk_legality(k, 0, 200, 40) if len(k.schedule) <= 800 else [],
    }
    if k.schedule:
        sim = ref.simulate(k)
        rec["sim"] = {"total": sim.total_cycles, "json": sim.to_json()}
    if rec["cands"]:
        rec["anneal"] = {}
        for cname, kw in CONFIGS.items():
            seeds = range(n_seeds) if cname == "default" else range(min(4, n_seeds))
            rec["anneal"][cname] = {
                str(s): anneal_record(k, ref.AnnealConfig(seed=s, **kw), full=s < 2) for s in seeds
            }
    return rec


def sample_records() -> list:
    out = []
    for seed in (0, 7, 123456789):
        for kind in ("int8", "int16", "int32"):
            for dist in ("uniform", "small", "zero"):
                plan = ref.TestPlan(
                    ret_ptr=1,
                    buffers=(ref.BufferSpec(0, 5, kind, dist), ref.BufferSpec(1, 3, "int32", "uniform")),
                    seed=seed,
                )
                for idx in (0, 1, 2, 25, 999999):
                    bufs = ref.difftest.sample_inputs(plan, idx)
                    out.append({"seed": seed, "kind": kind, "dist": dist, "index": idx,
                                "buf0": bufs[0].hex(), "buf1": bufs[1].hex()})
    return out


def main() -> None:
    listings = {}
    for name, text in corpus().items():
        big = len(text.splitlines()) > 400
        listings[name] = listing_record(name, text, n_seeds=4 if big else 16)
        print(f"{name}: n={listings[name]['n']} cands={len(listings[name]['cands'])}", flush=True)
    data = {"listings": listings, "samples": sample_records(),
            "generator": "tests/golden/make_golden.py", "reference": str(REF_SRC)}
    with gzip.open(OUT, "wt") as fh:
        json.dump(data, fh, sort_keys=True)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
