"""The C-ABI library loads without a GPU and exports every symbol include/sip.h declares."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_2403_16863_b200 import engine

ROOT = Path(__file__).resolve().parents[1]


def declared() -> list:
    text = (ROOT / "include" / "sip.h").read_text()
    return sorted(set(re.findall(r"^(?:const\s+)?\w+\*?\s+\*?(sip_\w+)\s*\(", text, re.M)))


def test_header_declares_the_abi():
    names = declared()
    assert "sip_anneal" in names and "sip_measure" in names and "sip_compare" in names
    assert len(names) >= 30


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(engine.LIB_PATH))
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_every_declared_symbol():
    assert set(declared()) <= set(engine._SIGS), set(declared()) - set(engine._SIGS)
    lib = engine.load_library()
    assert lib.sip_missing == ()
    assert lib.sip_version().decode().startswith("sip-b200")


def test_no_device_means_no_fallback(monkeypatch):
    """Without a GPU the engine refuses to run (no silent CPU path)."""
    lib = engine.load_library()
    n = ctypes.c_int32(-1)
    lib.sip_device_count(ctypes.byref(n))
    if n.value > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(engine.EngineUnavailable):
        engine.Context(0)


def test_cubin_frontend_parses_without_gpu():
    from paper_2403_16863_b200 import candidates
    from paper_2403_16863_b200.cubin import render_listing, schedule_perm
    from paper_2403_16863_b200.targets import TARGET_DIR

    L = render_listing((TARGET_DIR / "gemm_lrelu.cubin").read_bytes(), "gemm_lrelu_f16")
    assert L.n == len(L.words) and L.n > 500
    assert schedule_perm(L.kernel).tolist() == list(range(L.n))
    names = {ins.base_mnemonic for ins in L.kernel.schedule}
    assert {"UTCHMMA", "UTMALDG", "LDTM", "STG"} <= names  # tcgen05 + TMA evidence
    assert len(candidates(L.kernel)) >= 4
    assert L.pins.sum() > 0  # EXIT / MBARRIER offsets pinned
