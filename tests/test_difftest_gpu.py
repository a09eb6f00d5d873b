"""Differential testing on the GPU interpreter vs the reference's own verdicts
(tests/golden/make_golden_difftest.py ran the reference to produce them)."""
import gzip
import json
import time
from pathlib import Path

import pytest

from paper_2403_16863_b200 import parse_kernel
from paper_2403_16863_b200.difftest import (BufferSpec, TestPlan, first_failure_index, pass_curve,
                                            run_tests)
from paper_2403_16863_b200.interp import CompiledKernel, interpret

pytestmark = pytest.mark.gpu
G = json.load(gzip.open(Path(__file__).parent / "golden" / "difftest.json.gz", "rt"))


def plan_of(d, samples=64):
    return TestPlan(ret_ptr=d["ret_ptr"], samples=samples, seed=d.get("seed", 0),
                    buffers=tuple(BufferSpec(b["arg"], b["length"], b.get("kind", "int32"),
                                             b.get("dist", "uniform")) for b in d["buffers"]))


def test_verdicts_match_reference():
    for c in G["cases"]:
        v = run_tests(parse_kernel(c["ref"]), parse_kernel(c["mut"]), plan_of(c["plan"], c["samples"]),
                      fail_fast=c["fail_fast"])
        assert v.to_dict() == c["verdict"], c


def test_first_failure_indices_and_curve():
    ref = CompiledKernel(parse_kernel(G["base"]))
    plan = plan_of({"ret_ptr": 1, "buffers": [{"arg": 0, "length": 2}, {"arg": 1, "length": 4}]})
    got = [first_failure_index(ref, parse_kernel(t), plan, 2000) for t in G["mutants"]]
    assert got == G["first_failure"]
    curve = pass_curve(parse_kernel(G["base"]), [parse_kernel(t) for t in G["mutants"]], [1, 10, 100, 1000], plan)
    assert [list(x) for x in curve] == G["curve"]


def test_interpret_bindings_and_walked_mutants():
    for p in G["programs"]:
        k = parse_kernel(p["text"])
        for b in p["bindings"]:
            out = interpret(k, {0: bytes.fromhex(b["in0"]), 1: b"\x00" * 16}, ret_ptr=1)
            assert out.hex() == b["out"]
        plan = plan_of({"ret_ptr": 1, "seed": 3, "buffers": [{"arg": 0, "length": 4}, {"arg": 1, "length": 4}]},
                       200)
        for m in p["mutants"]:
            assert run_tests(k, parse_kernel(m["text"]), plan).to_dict() == m["verdict"], m


def test_inconclusive_paths():
    for c in G["inconclusive"]:
        v = run_tests(parse_kernel(c["ref"]), parse_kernel(c["mut"]), plan_of(c["plan"], c["samples"]))
        assert v.to_dict() == c["verdict"], c


def test_detection_curve_100k_samples():
    """Acceptance criterion 7 of the reference (test_acceptance.py:213-232), 100k samples."""
    t0 = time.perf_counter()
    plan = plan_of({"ret_ptr": 1, "buffers": [{"arg": 0, "length": 2}, {"arg": 1, "length": 4}]})
    muts = [parse_kernel(t) for t in G["mutants"]]
    curve = pass_curve(parse_kernel(G["base"]), muts, [1, 10, 100, 1_000, 10_000, 100_000], plan)
    counts = [n for _, n in curve]
    assert counts == sorted(counts, reverse=True) and counts[-1] == 10
    assert time.perf_counter() - t0 < 60.0


def test_million_sample_verdict_throughput():
    """A 1M-sample verdict on the reference's detection kernel (equivalent mutant)."""
    plan = plan_of({"ret_ptr": 1, "buffers": [{"arg": 0, "length": 2}, {"arg": 1, "length": 4}]}, 1_000_000)
    t0 = time.perf_counter()
    v = run_tests(parse_kernel(G["base"]), parse_kernel(G["mutants"][0]), plan)
    dt = time.perf_counter() - t0
    assert v.ok and v.passed == 1_000_000
    print(f"1M samples in {dt:.2f}s = {1e6 / dt:.0f} samples/s")


def test_fill_normal_statistics_and_streams():
    """sip_fill_normal: N(0, sigma^2) fp16, reproducible per (seed, stream), streams differ."""
    import ctypes

    import torch

    from paper_2403_16863_b200.engine import get_context

    ctx = get_context()
    n = 1 << 22
    a, b, c = (torch.empty(n, dtype=torch.float16, device="cuda") for _ in range(3))
    for t, stream in ((a, 5), (b, 5), (c, 6)):
        ctx.check(ctx.lib.sip_fill_normal(ctx.handle, ctypes.c_void_p(t.data_ptr()), n, 0, 11, stream, 0.5))
    torch.cuda.synchronize()
    assert torch.equal(a, b) and not torch.equal(a, c)
    x = a.float()
    assert abs(x.mean().item()) < 2e-3 and abs(x.std().item() - 0.5) < 5e-3
    assert x.abs().max().item() < 0.5 * 4.8  # 16-bit Box-Muller bound
    frac = (x.abs() < 0.5).float().mean().item()  # P(|z| < 1) = 0.6827
    assert abs(frac - 0.6827) < 3e-3
