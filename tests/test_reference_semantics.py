"""Host-side semantics the reference's own suite pins (no GPU needed):
annealing config/feedback/acceptance law (test_anneal.py), move vocabulary
(test_perturb.py), register/memory tables (test_deps.py), the external
measurement protocol (test_backends.py), the result store (test_store.py),
and schedule diffs (test_cli.py)."""
import json
import math
import os
import random
import stat
import textwrap

import pytest

from paper_2403_16863_b200 import (Action, AnnealConfig, Direction, ExternalCommandBackend,
                                   HistoryRecord, InvalidBaseline, MeasurementFailed, MoveRejected,
                                   NoCandidatesError, ResultStore, accept_move, apply_action,
                                   build_depgraph, candidates, feedback, input_hash, make_backend,
                                   mem_refs, parse_kernel, reads_writes, sample_action, swap_legal)
from paper_2403_16863_b200.cli import schedule_moves


def one(line):
    return parse_kernel(line + " ;\n").schedule[0]


class TestFeedbackAndConfig:
    def test_feedback_values(self):
        assert feedback(100.0, 100.0, 90.0) == pytest.approx(0.10, abs=0.0)
        assert feedback(100.0, 90.0, 90.0) == 0.0
        assert feedback(200.0, 180.0, 190.0) == pytest.approx(-0.05, abs=0.0)
        for t0 in (0.0, -1.0):
            with pytest.raises(InvalidBaseline):
                feedback(t0, 1.0, 1.0)

    def test_budget(self):
        assert AnnealConfig().iteration_budget == 95
        assert AnnealConfig(t_max=0.5, t_min=0.5).iteration_budget == 0
        for tmax, tmin, cool in [(2.0, 0.5, 1.1), (1.0, 0.001, 1.3), (8.0, 1.0, 2.0)]:
            cfg = AnnealConfig(t_max=tmax, t_min=tmin, cooling=cool)
            assert cfg.iteration_budget == math.ceil(math.log(tmax / tmin) / math.log(cool))

    @pytest.mark.parametrize("kw", [{"t_max": 0.0}, {"t_min": 0.0}, {"t_min": 2.0}, {"cooling": 1.0},
                                    {"measure_reps": 2}, {"tests_per_step": -1}])
    def test_rejects_bad_config(self, kw):
        with pytest.raises(ValueError):
            AnnealConfig(**kw)

    def test_temperature_sequence_is_repeated_division(self):
        cfg = AnnealConfig(cooling=1.05)
        t, temps = 1.0, cfg.temperatures()
        for i in range(cfg.iteration_budget):
            assert temps[i] == t
            t /= 1.05


class TestAcceptance:
    def test_downhill_never_consults_rng(self):
        class Blowup:
            def random(self):
                raise AssertionError("rng consulted on a downhill move")

        assert accept_move(-0.01, 0.5, Blowup())

    def test_boltzmann_rate(self):
        rng = random.Random(0)
        for de, temp in [(0.01, 0.05), (0.1, 0.1), (0.05, 0.01)]:
            n = 20000
            hits = sum(accept_move(de, temp, rng) for _ in range(n))
            assert abs(hits / n - math.exp(-de / temp)) < 0.03

    def test_history_record_json(self):
        r = HistoryRecord(3, 1, "up", None, 0.0, False, 0.5, rejected="boundary")
        assert json.loads(r.to_json()) == {"iteration": 3, "action": {"candidate": 1, "direction": "up"},
                                           "energy": None, "feedback": 0.0, "accepted": False,
                                           "temperature": 0.5, "rejected": "boundary"}


class TestMoves:
    STAGE = ("LDG.E R4, [R2.64] ;\nMOV R0, RZ ;\nLDG.E R5, [R2.64+0x4] ;\nMOV R1, RZ ;\n"
             "LDG.E R6, [R2.64+0x8] ;\nMOV R3, RZ ;\nLDG.E R7, [R2.64+0xc] ;\n")

    def test_action_encoding(self):
        class Fixed:
            def __init__(self, cell):
                self.cell = cell

            def randrange(self, n):
                assert n == 8
                return self.cell

        cset = candidates(parse_kernel(self.STAGE))
        assert sample_action(cset, Fixed(0)) == Action(0, Direction.UP)
        assert sample_action(cset, Fixed(1)) == Action(0, Direction.DOWN)
        assert sample_action(cset, Fixed(5)) == Action(2, Direction.DOWN)
        assert sample_action(cset, Fixed(7)) == Action(3, Direction.DOWN)

    def test_no_candidates(self):
        with pytest.raises(NoCandidatesError):
            sample_action(candidates(parse_kernel("MOV R0, RZ ;\n")), random.Random(0))

    def test_boundaries_and_dependencies(self):
        k = parse_kernel(self.STAGE)
        g = build_depgraph(k)
        with pytest.raises(MoveRejected) as e:
            apply_action(k, g, Action(0, Direction.UP))  # schedule edge
        assert e.value.reason == "boundary"
        moved = apply_action(k, g, Action(0, Direction.DOWN))  # independent MOV
        assert moved.schedule[1].base_mnemonic == "LDG"
        dep = parse_kernel("[B------:R-:W0:-:S01] LDG.E R4, [R2.64] ;\n[B0-----:R-:W-:-:S01] IADD3 R5, R4, 1, RZ ;\n")
        with pytest.raises(MoveRejected) as e:
            apply_action(dep, build_depgraph(dep), Action(0, Direction.DOWN))
        assert e.value.reason == "dependency"
        assert not swap_legal(build_depgraph(dep), dep, 0)

    def test_label_cut_blocks_move(self):
        k = parse_kernel("MOV R0, RZ ;\n.L_x_0:\nLDG.E R4, [R2.64] ;\n")
        with pytest.raises(MoveRejected) as e:
            apply_action(k, build_depgraph(k), Action(0, Direction.UP))
        assert e.value.reason == "boundary"


class TestDepsTables:
    RW = [
        ("LDG.E.128 R4, [R2.64+0x10]", {"R2", "R3"}, {"R4", "R5", "R6", "R7"}),
        ("STG.E.128 [R8.64], R4", {"R8", "R9", "R4", "R5", "R6", "R7"}, set()),
        ("IMAD.WIDE R18, R9, 0x80, R10", {"R9", "R10", "R11"}, {"R18", "R19"}),
        ("ISETP.GE.AND P0, PT, R4, 0x20, PT", {"R4"}, {"P0"}),
        ("@!P0 MOV R1, RZ", {"P0"}, {"R1"}),
        ("LDGSTS.E.BYPASS.128 [R219+0x4000], desc[UR16][R10.64], P0",
         {"R219", "R10", "R11", "UR16", "UR17", "P0"}, set()),
        ("ATOM.E.ADD R0, [R4.64], R2", {"R4", "R5", "R2"}, {"R0"}),
        ("XYZZY R1, R2", {"R1", "R2"}, {"R1", "R2"}),
    ]

    @pytest.mark.parametrize("line,r,w", RW, ids=[x[0] for x in RW])
    def test_reads_writes(self, line, r, w):
        rd, wr = reads_writes(one(line))
        assert set(rd) == r and set(wr) == w

    def test_mem_refs(self):
        (ref,) = mem_refs(one("LDG.E R0, [R2.64+0x10]"))
        assert (ref.space, ref.base, ref.offset, ref.size, ref.write) == ("global", "R2", 0x10, 4, False)
        sides = {(r.space, r.write) for r in mem_refs(one("LDGSTS.E.BYPASS.128 [R219+0x4000], desc[UR16][R10.64], P0"))}
        assert sides == {("shared", True), ("global", False)}
        assert mem_refs(one("IADD3 R6, R4, 0x10, RZ")) == ()


def _script(tmp_path, body: str) -> str:
    p = tmp_path / "adapter.sh"
    p.write_text("#!/bin/sh\n" + textwrap.dedent(body))
    p.chmod(p.stat().st_mode | stat.S_IEXEC)
    return str(p)


class TestExternalProtocol:
    def test_median_of_reps(self, tmp_path):
        counter = tmp_path / "n"
        counter.write_text("0")
        sh = _script(tmp_path, f"""
            n=$(cat {counter}); n=$((n+1)); echo $n > {counter}
            echo '{{"time_ms": '$n'.5}}'
        """)
        be = ExternalCommandBackend(f"{sh} {{schedule_file}}")
        s = be.measure(parse_kernel("MOV R0, RZ ;\n"), 5)
        assert s.value == 3.5 and s.raw == (1.5, 2.5, 3.5, 4.5, 5.5) and s.unit == "ms"

    def test_receives_exact_text(self, tmp_path):
        out = tmp_path / "seen.sass"
        sh = _script(tmp_path, f"""cp "$1" {out}; echo '{{"time_ms": 1}}'""")
        text = "[B------:R-:W-:-:S01] MOV R0, RZ ; // note\n"
        ExternalCommandBackend(f"{sh} {{schedule_file}}").measure(parse_kernel(text), 1)
        assert out.read_text() == text

    @pytest.mark.parametrize("body", ["exit 3", "echo nothing", "echo '{\"time_ms\": 1}'; echo '{\"time_ms\": 2}'",
                                      "echo '{\"time_ms\": -1}'"])
    def test_failures_raise(self, tmp_path, body):
        sh = _script(tmp_path, body)
        with pytest.raises(MeasurementFailed):
            ExternalCommandBackend(f"{sh} {{schedule_file}}").measure(parse_kernel("MOV R0, RZ ;\n"), 1)

    def test_timeout(self, tmp_path):
        sh = _script(tmp_path, "sleep 5")
        be = ExternalCommandBackend(f"{sh} {{schedule_file}}", timeout_s=0.2)
        with pytest.raises(MeasurementFailed):
            be.measure(parse_kernel("MOV R0, RZ ;\n"), 1)

    def test_factory(self):
        with pytest.raises(ValueError):
            make_backend("nonsense")
        with pytest.raises(ValueError):
            ExternalCommandBackend("no placeholder")
        assert make_backend("sim").unit == "cycles"


class TestStore:
    def test_best_pointer_only_advances(self, tmp_path):
        st = ResultStore(tmp_path)
        d = input_hash("x\r\n")
        assert d == input_hash("x\n")
        st.write_chain(d, 0, "A\n", "", {"passed": 1})
        m = st.update_manifest(d, baseline=10.0, unit="cycles", entries=[{"seed": 0, "time": 8.0, "passed": True,
                                                                           "iterations": 95}])
        assert m["best"]["seed"] == 0
        st.write_chain(d, 1, "B\n", "", {"passed": 1})
        m = st.update_manifest(d, baseline=10.0, unit="cycles", entries=[{"seed": 1, "time": 9.0, "passed": True,
                                                                           "iterations": 95}])
        assert m["best"]["seed"] == 0 and [e["seed"] for e in m["entries"]] == [0, 1]
        assert (st.run_dir(d) / "best.sass").read_text() == "A\n"
        assert not [p for p in os.listdir(st.run_dir(d)) if p.startswith(".tmp-")]


def test_schedule_moves_bubble_sort():
    a = parse_kernel("MOV R0, RZ ;\nMOV R1, RZ ;\nMOV R2, RZ ;\n")
    b = parse_kernel("MOV R2, RZ ;\nMOV R0, RZ ;\nMOV R1, RZ ;\n")
    assert schedule_moves(a, b) == [(1, 2), (0, 1)]
    with pytest.raises(ValueError):
        schedule_moves(a, parse_kernel("MOV R0, RZ ;\n"))
