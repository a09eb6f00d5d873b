"""Host frontend vs the reference: parse/serialize, classes, cuts, register and
memory facts -- checked listing by listing against goldens produced by the
reference itself (tests/golden/make_golden.py)."""
import pytest

from conftest import golden, listing_names
from paper_2403_16863_b200 import (ControlCode, ParseError, candidates, classify, mem_refs,
                                   parse_control, parse_kernel, reads_writes, serialize_kernel)
from paper_2403_16863_b200.ir import InstrClass
from paper_2403_16863_b200.sasstext import normalize_newlines

NAMES = listing_names()


@pytest.mark.parametrize("name", NAMES)
def test_round_trip(name):
    rec = golden()["listings"][name]
    k = parse_kernel(rec["text"], name=name)
    assert len(k.schedule) == rec["n"]
    assert (serialize_kernel(k) == normalize_newlines(rec["text"])) == rec["serialize_ok"]
    assert rec["serialize_ok"]


@pytest.mark.parametrize("name", NAMES)
def test_structure_matches_reference(name):
    rec = golden()["listings"][name]
    k = parse_kernel(rec["text"], name=name)
    assert list(k.block_boundaries) == rec["cuts"]
    assert list(candidates(k).positions) == rec["cands"]
    assert [ins.klass.value for ins in k.schedule] == rec["classes"]


@pytest.mark.parametrize("name", NAMES)
def test_register_sets_match_reference(name):
    rec = golden()["listings"][name]
    k = parse_kernel(rec["text"], name=name)
    for i, ins in enumerate(k.schedule):
        r, w = reads_writes(ins)
        assert [sorted(r), sorted(w)] == rec["rw"][i], (i, ins.source_text)


@pytest.mark.parametrize("name", NAMES)
def test_memory_refs_match_reference(name):
    rec = golden()["listings"][name]
    k = parse_kernel(rec["text"], name=name)
    for i, ins in enumerate(k.schedule):
        got = [[m.space, m.base, m.offset, m.size, int(m.write)] for m in mem_refs(ins)]
        assert got == rec["refs"][i], (i, ins.source_text)


def test_control_text_round_trip():
    for text in ("[B------:R-:W-:-:S01]", "[B0-2--5:R3:W1:Y:S15]", "B-1----:R-:W0:-:S00"):
        c = parse_control(text)
        assert c.to_text() == (text if text.startswith("[") else f"[{text}]")


@pytest.mark.parametrize("bad", ["[B------:R-:W-:-:S16]", "[B1-----:R-:W-:-:S01]",
                                 "[B------:R6:W-:-:S01]", "[B------]"])
def test_control_rejects_bad_fields(bad):
    with pytest.raises(ValueError):
        parse_control(bad)


def test_parse_error_on_bad_control():
    with pytest.raises(ParseError):
        parse_kernel("[B------:R-:W-:-:S99] MOV R0, RZ ;\n")


def test_classify_table():
    assert classify("LDG.E.128") is InstrClass.GLOBAL_LOAD
    assert classify("ldgsts.e.bypass.128") is InstrClass.GLOBAL_ASYNC_COPY
    assert classify("UTMALDG.2D") is InstrClass.OTHER  # K6: TMA is OTHER under reference rules
    assert classify("BAR.SYNC") is InstrClass.BARRIER
    assert ControlCode().to_text() == "[B------:R-:W-:-:S01]"


def test_cli_patch_roundtrip(tmp_path):
    """`patch` writes a cubin whose kernel section follows a listing's schedule: the
    identity listing reproduces the cubin, a swapped listing swaps the two 16-byte words."""
    from paper_2403_16863_b200.cli import main
    from paper_2403_16863_b200.cubin import Module, render_listing
    from paper_2403_16863_b200.ir import Kernel
    from paper_2403_16863_b200.sasstext import serialize_kernel
    from paper_2403_16863_b200.targets import TARGET_DIR

    cub = TARGET_DIR / "gemm_lrelu.cubin"
    L = render_listing(cub.read_bytes(), "gemm_lrelu_f16")
    ident = tmp_path / "ident.sass"
    ident.write_text(L.text)
    out = tmp_path / "out.cubin"
    assert main(["patch", str(cub), "gemm_lrelu_f16", str(ident), "-o", str(out)]) == 0
    m0 = Module(cub.read_bytes(), "gemm_lrelu_f16")
    m1 = Module(out.read_bytes(), "gemm_lrelu_f16")
    assert (m0.words() == m1.words()).all()
    sched = list(L.kernel.schedule)
    sched[10], sched[11] = sched[11], sched[10]
    sw = tmp_path / "swap.sass"
    sw.write_text(serialize_kernel(Kernel(name="k", schedule=tuple(sched))))
    assert main(["patch", str(cub), "gemm_lrelu_f16", str(sw), "-o", str(out)]) == 0
    w0, w1 = m0.words(), Module(out.read_bytes(), "gemm_lrelu_f16").words()
    assert (w1[10] == w0[11]).all() and (w1[11] == w0[10]).all() and (w1[12:] == w0[12:]).all()


@pytest.mark.parametrize("name,func", [("attn_fwd", "attn_fwd_f16"), ("gemm_lrelu", "gemm_lrelu_f16")])
def test_load_image_drops_debug_data_keeps_sass(name, func, tmp_path, monkeypatch):
    """The image the evaluator loads has the -lineinfo debug data removed (the driver's
    per-load cost grows with it) and byte-identical SASS."""
    import ctypes
    import re
    import shutil
    import subprocess

    from paper_2403_16863_b200.engine import load_library
    from paper_2403_16863_b200.targets import TARGET_DIR

    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not available")
    lib = load_library()
    data = (TARGET_DIR / f"{name}.cubin").read_bytes()
    m = ctypes.c_void_p()
    assert lib.sip_module_open(None, data, len(data), func.encode(), ctypes.byref(m)) == 0
    monkeypatch.setenv("SIP_PATCH_LOAD_IMAGE", "1")
    size = ctypes.c_size_t()
    assert lib.sip_module_patch(m, None, None, ctypes.byref(size)) == 0
    buf = ctypes.create_string_buffer(size.value)
    assert lib.sip_module_patch(m, None, buf, ctypes.byref(size)) == 0
    lib.sip_module_close(m)
    assert size.value < len(data) * 0.5
    out = tmp_path / "load.cubin"
    out.write_bytes(buf.raw[: size.value])

    def sass(path):
        text = subprocess.run(["cuobjdump", "-sass", str(path)], capture_output=True, text=True, check=True).stdout
        return [ln for ln in text.splitlines() if re.match(r"\s+/\*[0-9a-f]{4}\*/", ln)]

    assert sass(out) == sass(TARGET_DIR / f"{name}.cubin")
