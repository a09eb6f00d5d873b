"""Goldens for differential testing, produced by running the reference.

    python tests/golden/make_golden_difftest.py   # writes tests/golden/difftest.json.gz

Records run_tests verdicts (both fail_fast settings), first_failure_index,
pass_curve, interpret() outputs on explicit bindings, and the verdicts of the
reference's inconclusive paths, for the reference's own test kernels
(kernels.BASE_DETECT with its labelled mutants, kernels.random_program) and a
few walked mutants.  Texts are stored with the results.
"""
from __future__ import annotations

import gzip
import json
import random
import struct
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import kernels as refk  # noqa: E402
import sasstune as ref  # noqa: E402
from sasstune.difftest import BufferSpec, TestPlan, first_failure_index, pass_curve, run_tests  # noqa: E402
from sasstune.machine import CompiledKernel, interpret  # noqa: E402

OUT = Path(__file__).with_name("difftest.json.gz")
DETECT = {"ret_ptr": 1, "buffers": [{"arg": 0, "length": 2}, {"arg": 1, "length": 4}], "seed": 0}


def plan_of(d, samples=64):
    return TestPlan(ret_ptr=d["ret_ptr"],
                    buffers=tuple(BufferSpec(b["arg"], b["length"], b.get("kind", "int32"),
                                             b.get("dist", "uniform")) for b in d["buffers"]),
                    samples=samples, seed=d.get("seed", 0))


def walk(kernel, seed, steps, unsafe):
    rng = random.Random(seed)
    k = kernel
    g = ref.build_depgraph(k)
    for _ in range(steps):
        a = ref.sample_action(ref.candidates(k), rng)
        try:
            k = ref.apply_action(k, g, a, unsafe=unsafe)
        except ref.MoveRejected:
            continue
        g = ref.build_depgraph(k)
    return ref.serialize_kernel(k)


def main():
    base = refk.BASE_DETECT
    mutants = refk.detect_equivalents() + [t for t, _ in refk.detect_violators()]
    cases = []
    for j, mt in enumerate(mutants):
        for samples in (64, 300):
            for ff in (False, True):
                v = run_tests(ref.parse_kernel(base), ref.parse_kernel(mt), plan_of(DETECT, samples), fail_fast=ff)
                cases.append({"ref": base, "mut": mt, "plan": DETECT, "samples": samples, "fail_fast": ff,
                              "verdict": v.to_dict()})
    ck = CompiledKernel(ref.parse_kernel(base))
    ffi = [first_failure_index(ck, ref.parse_kernel(t), plan_of(DETECT), 2000) for t in mutants]
    curve = pass_curve(ref.parse_kernel(base), [ref.parse_kernel(t) for t in mutants], [1, 10, 100, 1000],
                       plan_of(DETECT))

    # random programs: explicit bindings and walked mutants (safe and unsafe)
    progs = []
    plan_rp = {"ret_ptr": 1, "buffers": [{"arg": 0, "length": 4}, {"arg": 1, "length": 4}], "seed": 3}
    for seed in range(12):
        text, _ = refk.random_program(seed, n_ops=10)
        k = ref.parse_kernel(text)
        binds = []
        for j in range(3):
            gen = random.Random(f"case:{seed}:{j}")
            buffers = {0: struct.pack("<4I", *(gen.getrandbits(32) for _ in range(4))), 1: b"\x00" * 16}
            binds.append({"in0": buffers[0].hex(), "out": interpret(k, buffers, ret_ptr=1).hex()})
        muts = []
        for w, unsafe in ((0, False), (1, True), (2, True)):
            mt = walk(k, 100 * seed + w, 12, unsafe)
            v = run_tests(k, ref.parse_kernel(mt), plan_of(plan_rp, 200))
            muts.append({"text": mt, "unsafe": unsafe, "verdict": v.to_dict()})
        progs.append({"text": text, "bindings": binds, "mutants": muts})

    # inconclusive paths
    loopy = "BRA 0x10 ;\nEXIT ;\n"
    pipe = (Path("/root/reference/pkg/tests/data") / "pipeline.sass").read_text()
    bad_ref = pipe.replace("[R2.64+0x4]", "[R2.64+0x400]")
    small = {"ret_ptr": 1, "buffers": [{"arg": 0, "length": 2}, {"arg": 1, "length": 1}], "seed": 0}
    inconc = [
        {"ref": base, "mut": loopy, "plan": DETECT, "samples": 64,
         "verdict": run_tests(ref.parse_kernel(base), ref.parse_kernel(loopy), plan_of(DETECT)).to_dict()},
        {"ref": loopy, "mut": base, "plan": DETECT, "samples": 64,
         "verdict": run_tests(ref.parse_kernel(loopy), ref.parse_kernel(base), plan_of(DETECT)).to_dict()},
        {"ref": bad_ref, "mut": pipe, "plan": small, "samples": 4,
         "verdict": run_tests(ref.parse_kernel(bad_ref), ref.parse_kernel(pipe), plan_of(small, 4)).to_dict()},
        {"ref": pipe, "mut": bad_ref, "plan": small, "samples": 4,
         "verdict": run_tests(ref.parse_kernel(pipe), ref.parse_kernel(bad_ref), plan_of(small, 4)).to_dict()},
    ]
    data = {"cases": cases, "first_failure": ffi, "mutants": mutants, "base": base, "curve": curve,
            "programs": progs, "inconclusive": inconc}
    with gzip.open(OUT, "wt") as fh:
        json.dump(data, fh, sort_keys=True)
    print("wrote", OUT, OUT.stat().st_size, "first_failure", ffi, "curve", curve)


if __name__ == "__main__":
    main()
