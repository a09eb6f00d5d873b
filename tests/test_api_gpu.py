"""Public surface end to end on the GPU: CLI, config, store, estimator (reference
cli.py / store.py / estimator.py behaviours, incl. the README hide.sass run)."""
import json

import pytest

from paper_2403_16863_b200 import ScheduleTuner, parse_kernel
from paper_2403_16863_b200.cli import main

pytestmark = pytest.mark.gpu

HIDE = (
    "[B------:R-:W-:-:S08] IADD3 R20, RZ, 0x1, RZ ;\n[B------:R-:W-:-:S08] IADD3 R21, RZ, 0x1, RZ ;\n"
    "[B------:R-:W-:-:S08] IADD3 R22, RZ, 0x1, RZ ;\n[B------:R-:W-:-:S08] IADD3 R23, RZ, 0x1, RZ ;\n"
    "[B------:R-:W0:-:S01] LDG.E R4, [R2.64] ;\n[B0-----:R-:W-:-:S01] IADD3 R5, R4, 0x1, RZ ;\n"
)


def test_optimize_report_and_store(tmp_path, capsys):
    f = tmp_path / "hide.sass"
    f.write_text(HIDE)
    rc = main(["optimize", str(f), "--store", str(tmp_path / "store")])
    out = capsys.readouterr().out.splitlines()
    assert rc == 0
    assert out[0] == "input: hide  instructions: 6  candidates: 1"
    assert out[1] == "baseline: 436 cycles"
    assert out[2] == "chain seed=0: best 404 cycles after 95 iterations, tests skipped"
    assert out[3] == "best: 404 cycles (seed 0), improvement 7.34%"
    store_dir = out[4].split(": ", 1)[1]
    best = (tmp_path / "store" / store_dir.split("/")[-1] / "best.sass").read_text()
    assert best.splitlines()[0] == "[B------:R-:W0:-:S01] LDG.E R4, [R2.64] ;"
    manifest = json.loads((tmp_path / "store" / store_dir.split("/")[-1] / "manifest.json").read_text())
    assert manifest["best"]["time"] == 404.0


def test_exit_codes(tmp_path, capsys):
    alu = tmp_path / "alu.sass"
    alu.write_text("MOV R0, RZ ;\nMOV R1, RZ ;\n")
    assert main(["optimize", str(alu)]) == 3
    bad = tmp_path / "bad.sass"
    bad.write_text("[B------:R-:W-:-:S99] MOV R0, RZ ;\n")
    assert main(["optimize", str(bad)]) == 2
    h = tmp_path / "h.sass"
    h.write_text(HIDE)
    assert main(["optimize", str(h), "--backend", "nope"]) == 4
    assert main(["verify", str(h), str(h)]) == 1


def test_simulate_and_diff(tmp_path, capsys):
    a = tmp_path / "a.sass"
    a.write_text(HIDE)
    lines = HIDE.splitlines()
    b = tmp_path / "b.sass"
    b.write_text("\n".join([lines[4]] + lines[:4] + [lines[5]]) + "\n")
    assert main(["simulate", str(a)]) == 0
    assert json.loads(capsys.readouterr().out)["total_cycles"] == 436
    assert main(["diff", str(a), str(b)]) == 0
    moves = json.loads(capsys.readouterr().out)["moves"]
    assert moves == [{"swap": [3, 4]}, {"swap": [2, 3]}, {"swap": [1, 2]}, {"swap": [0, 1]}]


def test_estimator_fit_transform():
    t = ScheduleTuner(chains=3)
    out = t.fit_transform(HIDE)
    assert t.best_time_ == 404.0 and t.n_iterations_ == 285
    assert parse_kernel(out).schedule[0].base_mnemonic == "LDG"
    with pytest.raises(ValueError):
        t.transform("MOV R0, RZ ;\n")


def test_b200_external_adapter(tmp_path):
    """The reference's external protocol priced on the B200: ExternalCommandBackend
    (backends.py:73-116) spawns `sip measure`, which prints one {"time_ms": x} line."""
    import sys

    from paper_2403_16863_b200 import serialize_kernel
    from paper_2403_16863_b200.backends import ExternalCommandBackend, MeasurementFailed
    from paper_2403_16863_b200.cubin import render_listing
    from paper_2403_16863_b200.ir import Kernel
    from paper_2403_16863_b200.targets import TARGET_DIR

    listing = render_listing((TARGET_DIR / "gemm_lrelu.cubin").read_bytes(), "gemm_lrelu_f16")
    cmd = (f"{sys.executable} -m paper_2403_16863_b200 measure --target gemm "
           "--shape M=512,N=512,K=2048 --reps 3 {schedule_file}")
    from pathlib import Path

    be = ExternalCommandBackend(cmd, timeout_s=300, workdir=str(Path(__file__).resolve().parents[1]))
    s = be.measure(listing.kernel, reps=1)
    assert s.unit == "ms" and 0.0 < s.value < 5.0
    # a schedule that is not a permutation of the cubin is a measurement failure
    sched = list(listing.kernel.schedule)
    bad = Kernel(name="bad", schedule=tuple(sched[:-1] + [sched[0]]))
    with pytest.raises(MeasurementFailed):
        be.measure(bad, reps=1)
    f = tmp_path / "x.sass"
    f.write_text(serialize_kernel(listing.kernel))
    assert main(["measure", str(f), "--shape", "M=512,N=512,K=2048", "--reps", "2"]) == 0


def test_optimize_b200_emits_patched_cubin(tmp_path, capsys):
    """`optimize --backend b200:gemm` on the decoded listing of the shipped cubin: the
    store gets best.sass and best.cubin, whose kernel words are a permutation of the
    original's (the emitted schedule as a loadable binary)."""
    import numpy as np

    from paper_2403_16863_b200.cubin import Module
    from paper_2403_16863_b200.targets import TARGET_DIR

    cub = TARGET_DIR / "gemm_lrelu.cubin"
    lst = tmp_path / "gemm.sass"
    assert main(["decode", str(cub), "gemm_lrelu_f16", "-o", str(lst)]) == 0
    rc = main(["optimize", str(lst), "--backend", "b200:gemm", "--chains", "2", "--store", str(tmp_path / "st")])
    out = capsys.readouterr().out
    assert rc == 0, out
    run = [p for p in (tmp_path / "st").iterdir() if p.is_dir()][0]
    assert (run / "best.sass").exists() and (run / "best.cubin").exists()
    w0 = Module(cub.read_bytes(), "gemm_lrelu_f16").words()
    w1 = Module((run / "best.cubin").read_bytes(), "gemm_lrelu_f16").words()
    key = lambda w: sorted(map(tuple, w.tolist()))  # noqa: E731
    assert key(w0) == key(w1)
