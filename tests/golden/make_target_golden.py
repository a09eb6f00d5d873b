"""Reference-run goldens for the decoded sm_100a tuning-target listings.

    python tests/golden/make_target_golden.py        # writes tests/golden/targets.json.gz

The listings under ``tests/golden/listings/`` are the cubin frontend's output
for the shipped ``gemm_lrelu_f16`` (n = 1 184) and ``attn_fwd_f16`` targets:
exactly what ``bench.py`` searches.  This script runs the *reference*
(``/root/reference/pkg/src/sasstune``, importable only in this container) on
them: register/memory facts, cuts, candidates, the simulate() report, legality
along a thinned random walk (every adjacent slot at each sampled point; the
big listings make a dense walk take minutes), and full annealing histories
(``anneal.anneal`` with ``SimulatorBackend``, ``anneal.py:123-213``) for the
default, ``long``, ``unsafe`` and ``hot`` configurations.  One process per
(listing, config, seed): the reference takes ~10 s (GEMM) to ~30 s
(attention) per default chain.
"""
from __future__ import annotations

import gzip
import json
import sys
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

import make_golden as mg  # noqa: E402  (imports the reference)
from make_golden import CONFIGS, anneal_record, ref, walk_legality  # noqa: E402

OUT = HERE / "targets.json.gz"
LISTINGS = HERE / "listings"
SEEDS = {"default": range(8), "long": range(2), "unsafe": range(2), "hot": range(2)}
SEEDS_BIG = {"default": range(4), "long": range(2), "unsafe": range(2), "hot": range(2)}


def _anneal_job(name: str, text: str, cname: str, seed: int):
    k = ref.parse_kernel(text, name=name)
    return name, cname, seed, anneal_record(k, ref.AnnealConfig(seed=seed, **CONFIGS[cname]), full=True)


def _facts_job(name: str, text: str):
    k = ref.parse_kernel(text, name=name)
    mach = ref.MachineConfig()
    rw = [mg.reads_writes(ins) for ins in k.schedule]
    sim = ref.simulate(k)
    return name, {
        "text": text,
        "n": len(k.schedule),
        "rw": [[sorted(r), sorted(w)] for r, w in rw],
        "refs": [[[m.space, m.base, m.offset, m.size, int(m.write)] for m in mg.mem_refs(ins)]
                 for ins in k.schedule],
        "cuts": list(k.block_boundaries),
        "cands": list(ref.candidates(k).positions),
        "classes": [ins.klass.value for ins in k.schedule],
        "serialize_ok": ref.serialize_kernel(k) == ref.sasstext.normalize_newlines(text),
        "walks": walk_legality(k, 0, 60, 6),
        "sim": {"total": sim.total_cycles, "json": sim.to_json()},
        # what the oracle's own table builder needs (oracle/golden_tables.py), straight from
        # the reference: scoreboard fields (ir.ControlCode) and machine.py latencies
        "ctrl": [[sorted(c.wait_mask), c.read_barrier, c.write_barrier, c.stall_cycles]
                 if c is not None else None for c in (ins.control for ins in k.schedule)],
        "lat": [mach.latency_of(ins) for ins in k.schedule],
    }


def refresh_facts() -> None:
    """Recompute the per-listing facts only, keeping the (slow) annealing records."""
    with gzip.open(OUT, "rt") as fh:
        data = json.load(fh)
    for name, rec in data["listings"].items():
        _, facts = _facts_job(name, rec["text"])
        facts["anneal"] = rec["anneal"]
        data["listings"][name] = facts
    with gzip.open(OUT, "wt") as fh:
        json.dump(data, fh, sort_keys=True)
    print(f"refreshed facts in {OUT}")


def main() -> None:
    if "--facts-only" in sys.argv:
        refresh_facts()
        return
    texts = {p.stem: p.read_text() for p in sorted(LISTINGS.glob("*.sass"))}
    out = {}
    with ProcessPoolExecutor(8) as ex:
        facts = [ex.submit(_facts_job, n, t) for n, t in texts.items()]
        jobs = []
        for n, t in texts.items():
            seeds = SEEDS_BIG if t.count("\n") > 2000 else SEEDS
            for cname, rs in seeds.items():
                jobs += [ex.submit(_anneal_job, n, t, cname, s) for s in rs]
        for f in facts:
            n, rec = f.result()
            rec["anneal"] = {c: {} for c in CONFIGS}
            out[n] = rec
            print(f"{n}: n={rec['n']} cands={len(rec['cands'])}", flush=True)
        for f in jobs:
            n, cname, seed, rec = f.result()
            out[n]["anneal"][cname][str(seed)] = rec
            print(f"  {n} {cname} seed {seed}: priced {rec['priced']} best {rec['best_energy']}", flush=True)
    data = {"listings": out, "generator": "tests/golden/make_target_golden.py",
            "reference": str(mg.REF_SRC)}
    with gzip.open(OUT, "wt") as fh:
        json.dump(data, fh, sort_keys=True)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
