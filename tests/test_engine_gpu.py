"""CUDA search engine (G1 legality, G2 annealing, scoreboard) vs reference goldens
and vs the CPU oracle.  Bit-exact: histories compared as JSONL bytes."""
import hashlib

import numpy as np
import pytest

from conftest import golden, listing_names
from golden_configs import CONFIGS
from golden.edge_listings import EDGE_LISTINGS
from oracle import oracle
from paper_2403_16863_b200 import (AnnealConfig, SimulatorBackend, anneal, parse_kernel, run_search,
                                   simulate)
from paper_2403_16863_b200.anneal import anneal_batch_sim
from paper_2403_16863_b200.engine import get_context
from paper_2403_16863_b200.machine import MachineConfig
from paper_2403_16863_b200.tables import KernelTables

pytestmark = pytest.mark.gpu

ANNEAL_NAMES = listing_names(lambda r: "anneal" in r)
SIM_NAMES = listing_names(lambda r: "sim" in r)
WALK_NAMES = listing_names(lambda r: r["walks"])


def setup(name):
    rec = golden()["listings"][name]
    k = parse_kernel(rec["text"], name=name)
    t = KernelTables.build(k, MachineConfig())
    return rec, k, t, get_context().kernel(t)


@pytest.mark.parametrize("name", SIM_NAMES)
def test_simulate_report_matches_reference(name):
    rec, k, t, dk = setup(name)
    assert simulate(k).to_json() == rec["sim"]["json"]


@pytest.mark.parametrize("name", WALK_NAMES)
def test_legality_matches_reference_walks(name):
    rec, k, t, dk = setup(name)
    n = t.n
    for w in rec["walks"]:
        los = np.arange(n - 1, dtype=np.int32)
        scheds = np.tile(np.asarray(w["perm"], dtype=np.uint16), (n - 1, 1))
        assert dk.legality(scheds, los).tolist() == w["legal"]


@pytest.mark.parametrize("name", ANNEAL_NAMES)
def test_anneal_histories_byte_identical(name):
    rec, k, t, dk = setup(name)
    for cname, runs in rec["anneal"].items():
        cfg = AnnealConfig(**CONFIGS[cname])
        seeds = [int(s) for s in runs]
        states = anneal_batch_sim(k, MachineConfig(), cfg, seeds, tables=t)
        for seed, st in zip(seeds, states):
            want = runs[str(seed)]
            jsonl = st.history_jsonl()
            if "jsonl" in want:
                assert jsonl == want["jsonl"], (cname, seed)
            assert hashlib.sha256(jsonl.encode()).hexdigest() == want["sha256"], (cname, seed)
            assert st.best_perm.tolist() == want["best"]
            assert st.best_energy == want["best_energy"]
            assert st.current_energy == want["current_energy"]
            assert st.baseline == want["baseline"]
            assert st.ambiguous == 0


def test_public_anneal_api_single_chain():
    rec, k, t, dk = setup("hide")
    st = anneal(k, SimulatorBackend(), AnnealConfig(seed=0))
    assert st.baseline == 436.0 and st.best_time == 404.0 and st.iterations == 95
    assert st.history_jsonl() == rec["anneal"]["default"]["0"]["jsonl"]


class _PythonPricedSim(SimulatorBackend):
    """Same energy as SimulatorBackend but priced through measure() -> step mode."""

    def measure(self, kernel, reps=1):
        return super().measure(kernel, reps)


@pytest.mark.parametrize("name", ["copy_stage_a", "pipeline", "base_detect", "random_program_2"])
def test_step_mode_matches_reference(name):
    rec, k, t, dk = setup(name)
    for seed in (0, 1):
        st = anneal(k, _PythonPricedSim(), AnnealConfig(seed=seed))
        want = rec["anneal"]["default"][str(seed)]
        assert hashlib.sha256(st.history_jsonl().encode()).hexdigest() == want["sha256"]


@pytest.mark.parametrize("name", ["synthetic_mix_0", "synthetic_mix_1", "random_program_0", "corridor"])
@pytest.mark.parametrize("cname", ["default", "long"])
def test_many_chains_vs_oracle(name, cname):
    """Hundreds of seeds beyond the goldens: device records == oracle records."""
    rec, k, t, dk = setup(name)
    cfg = AnnealConfig(**CONFIGS[cname])
    temps = cfg.temperatures()
    seeds = np.arange(1000, 1000 + (256 if cname == "default" else 64), dtype=np.int64)
    hist, best, cur, summ = dk.anneal(seeds, temps)
    ol = oracle.OracleListing(t)
    for c, s in enumerate(seeds):
        oh, ob, oc, os_ = ol.anneal(int(s), temps)
        assert np.array_equal(hist[c], oh), (name, int(s))
        assert np.array_equal(best[c], ob) and np.array_equal(cur[c], oc)
        assert summ["best_energy"][c] == os_["best_energy"]
    assert int(summ["ambiguous"].sum()) == 0


def test_run_search_batched_ranking():
    rec, k, t, dk = setup("hide")
    rep = run_search(k, SimulatorBackend(), AnnealConfig(seed=0), chains=8)
    assert [o.seed for o in rep.chains] == list(range(8))
    assert rep.best_time == 404.0 and rep.best.seed == 0
    assert rep.baseline == 436.0


def test_device_sample_stream_matches_reference():
    """sip_sample_inputs: CPython Random(f"{seed}:{index}") streams generated on the device."""
    import ctypes

    ctx = get_context()
    kinds = {"int8": 1, "int16": 2, "int32": 4}
    dists = {"uniform": 0, "small": 1, "zero": 2}
    for rec in golden()["samples"]:
        c0 = kinds[rec["kind"]]
        nbytes = np.array([5 * c0, 12], dtype=np.int32)
        cell = np.array([c0, 4], dtype=np.int32)
        dist = np.array([dists[rec["dist"]], 0], dtype=np.int32)
        out = np.zeros(int(nbytes.sum()), dtype=np.uint8)
        P = ctypes.POINTER(ctypes.c_int32)
        ctx.check(ctx.lib.sip_sample_inputs(ctx.handle, rec["seed"], rec["index"], 1, 2,
                                            nbytes.ctypes.data_as(P), cell.ctypes.data_as(P),
                                            dist.ctypes.data_as(P),
                                            out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))))
        assert out[: nbytes[0]].tobytes().hex() == rec["buf0"], rec
        assert out[nbytes[0]:].tobytes().hex() == rec["buf1"], rec


def test_anneal_epoch_restart_matches_oracle_from_identity():
    """sip_anneal_ex with start=identity is the plain chain (the epoch-restart path)."""
    rec, k, t, dk = setup("synthetic_mix_2")
    temps = AnnealConfig().temperatures()
    seeds = np.arange(500, 628, dtype=np.int64)
    hist, summ, champ, w = dk.anneal_epoch(seeds, temps, start=np.arange(t.n, dtype=np.uint16))
    ol = oracle.OracleListing(t)
    best_e = []
    for c, s in enumerate(seeds):
        oh, ob, _, os_ = ol.anneal(int(s), temps)
        assert np.array_equal(hist[c], oh)
        best_e.append((os_["best_energy"], int(s), ob))
    e, s, ob = min(best_e, key=lambda x: (x[0], x[1]))
    assert seeds[w] == s and np.array_equal(champ, ob)


def test_anneal_epoch_reduced_matches_oracle_champion():
    """sip_anneal_epoch: device seeds seed_base + c, champion and sums reduced on the
    device, equal to the oracle's chains ranked like driver.py:81-85."""
    rec, k, t, dk = setup("synthetic_mix_2")
    temps = AnnealConfig().temperatures()
    res, champ = dk.anneal_epoch_reduced(700, 96, temps)
    ol = oracle.OracleListing(t)
    best_e, priced = [], 0
    for s in range(700, 796):
        oh, ob, _, os_ = ol.anneal(s, temps)
        best_e.append((os_["best_energy"], s, ob))
        priced += int((oh["status"] <= 1).sum())
    e, s, ob = min(best_e, key=lambda x: (x[0], x[1]))
    assert res["best_seed"] == s and res["champion_chain"] == s - 700
    assert res["best_energy"] == e and np.array_equal(champ, ob)
    assert res["priced"] == priced and res["ambiguous"] == 0


def test_pinned_summary_pool_recycles_blocks():
    """Chain summaries land in page-locked blocks that are reused once every view is gone,
    and a block stays valid while any view of it is alive."""
    import gc

    from paper_2403_16863_b200.engine import SUMMARY_DTYPE, pinned_pool

    pool = pinned_pool(get_context().lib)
    a = pool.records(1000, SUMMARY_DTYPE)
    addr = a.ctypes.data
    a["t0"] = 3.5
    view = a["t0"][10:]
    del a
    gc.collect()
    b = pool.records(1000, SUMMARY_DTYPE)
    addr_b = b.ctypes.data
    assert addr_b != addr  # the first block is still held by `view`
    assert float(view[0]) == 3.5
    del view, b
    gc.collect()
    # both blocks are back in the pool: the next two requests reuse them
    c = pool.records(1000, SUMMARY_DTYPE)
    d = pool.records(1000, SUMMARY_DTYPE)
    assert {c.ctypes.data, d.ctypes.data} == {addr, addr_b}


def test_anneal_wave_is_whole_blocks_on_every_sm():
    """sip_anneal_wave: chains of one full wave of the fused kernel (128-thread blocks,
    at least one resident per SM)."""
    from bench import decoded_listing

    listing = decoded_listing()
    dk = get_context().kernel(KernelTables.build(listing.kernel, MachineConfig()))
    wave = dk.wave_chains()
    sms = get_context().sm_count
    assert wave > 0 and wave % (128 * sms) == 0
    assert wave // (128 * sms) <= 16  # 2 048 threads per SM at most


# edge-case listings (boundaries, no legal move, cuts, all-candidate, tiny): pinned to
# the reference by tests/golden/edge.json; the device chains must equal the oracle


@pytest.mark.parametrize("name", sorted(EDGE_LISTINGS))
def test_edge_listings_vs_oracle(name):
    k = parse_kernel(EDGE_LISTINGS[name], name=name)
    t = KernelTables.build(k, MachineConfig())
    dk = get_context().kernel(t)
    ol = oracle.OracleListing(t)
    for cname in ("default", "unsafe", "long"):
        cfg = AnnealConfig(**CONFIGS[cname])
        temps = cfg.temperatures()
        seeds = np.arange(64, dtype=np.int64)
        hist, best, cur, summ = dk.anneal(seeds, temps, unsafe=cfg.unsafe_moves)
        for c, s in enumerate(seeds):
            oh, ob, oc, os_ = ol.anneal(int(s), temps, unsafe=cfg.unsafe_moves)
            assert np.array_equal(hist[c], oh), (name, cname, int(s))
            assert np.array_equal(best[c], ob) and np.array_equal(cur[c], oc)
            assert summ["best_energy"][c] == os_["best_energy"]


def _edge_golden():
    import json
    from pathlib import Path

    return json.loads((Path(__file__).parent / "golden" / "edge.json").read_text())


@pytest.mark.parametrize("name", sorted(EDGE_LISTINGS))
def test_edge_listings_public_api_matches_reference(name):
    """The public anneal() on the edge listings, fused (SimulatorBackend) and step mode
    (priced through measure()), reproduces the reference's histories and schedules."""
    want_all = _edge_golden()[name]["anneal"]
    k = parse_kernel(EDGE_LISTINGS[name], name=name)
    for cname in ("default", "unsafe", "long"):
        for seed in (0, 1, 2, 3):
            want = want_all[cname][str(seed)]
            for backend in (SimulatorBackend(), _PythonPricedSim()):
                st = anneal(k, backend, AnnealConfig(seed=seed, **CONFIGS[cname]))
                assert hashlib.sha256(st.history_jsonl().encode()).hexdigest() == want["sha256"], \
                    (cname, seed, type(backend).__name__)


def test_no_candidates_raises_like_the_reference():
    from paper_2403_16863_b200.perturb import NoCandidatesError

    k = parse_kernel("[B------:R-:W-:-:S04] IADD3 R5, R6, 0x1, RZ ;\n"
                     "[B------:R-:W-:-:S04] IADD3 R8, R9, 0x1, RZ ;\n", name="alu_only")
    with pytest.raises(NoCandidatesError):
        run_search(k, SimulatorBackend(), AnnealConfig(seed=0), chains=4)


@pytest.mark.parametrize("name", ["gemm_lrelu_f16", "random_program_3", "corridor", "base_detect"])
def test_slot_chains_equal_dense_rows(name, monkeypatch):
    """SlotRow chains (candidate slots in shared memory, rows built on read) and dense-row
    chains (SIP_NO_SLOTS=1) are the same search: histories, best and current schedules and
    summaries are identical for the same seeds, on the decoded GEMM target listing (k = 5)
    and on golden listings with 4-8 candidates."""
    from pathlib import Path

    if name == "gemm_lrelu_f16":
        text = (Path(__file__).parent / "golden" / "listings" / f"{name}.sass").read_text()
    else:
        text = golden()["listings"][name]["text"]
    k = parse_kernel(text, name=name)
    t = KernelTables.build(k, MachineConfig())
    assert 0 < len(t.global_ids) <= 8  # a SlotRow listing
    dk = get_context().kernel(t)
    temps = AnnealConfig().temperatures()
    seeds = np.arange(5_000, 5_000 + 2_048, dtype=np.int64)
    slots = dk.anneal(seeds, temps)
    monkeypatch.setenv("SIP_NO_SLOTS", "1")
    dense = dk.anneal(seeds, temps)
    for a, b in zip(slots, dense):
        assert np.array_equal(a, b)
