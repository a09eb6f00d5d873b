"""Interpreter compile rules (no GPU needed): the supported subset and the
refusals follow the reference's closure compiler (machine.py:407-654)."""
import pytest

from paper_2403_16863_b200 import parse_kernel
from paper_2403_16863_b200.interp import (CompiledKernel, UnsupportedInstruction, buffer_bases,
                                          compile_kernel)

from conftest import golden


@pytest.mark.parametrize("line", [
    "BRA 0x10", "IMAD.HI R1, R2, R3, R4", "IADD3 R1, P0, PT, R2, R3, RZ", "RED.E.ADD [R2.64], R4",
    "LDG.E R0, desc[UR4][R2.64]", "MOV R1, R2, 0x3", "FFMA R1, R2, R3, R4", "ISETP.GE.EX.AND P0, PT, R1, R2, PT",
    "SHF.L.R.U32 R1, R2, 0x1, R3", "LOP3 R1, R2, R3, R4, 0xc0", "IADD3 R1, R2, 1.5, RZ",
])
def test_unsupported_is_refused_at_compile_time(line):
    with pytest.raises(UnsupportedInstruction):
        CompiledKernel(parse_kernel(line + " ;\n"))


def test_reference_programs_compile():
    for name in ("base_detect", "interp_hide", "pipeline") + tuple(f"random_program_{i}" for i in range(6)):
        k = parse_kernel(golden()["listings"][name]["text"])
        prog = compile_kernel(k, {0: 16, 1: 16})
        assert len(prog) >= 1


def test_buffer_layout_is_the_reference_layout():
    assert buffer_bases({1: 16, 0: 8}) == {0: 0x10000, 1: 0x10000 + 256 + 256}
    assert buffer_bases({0: 300}) == {0: 0x10000}
