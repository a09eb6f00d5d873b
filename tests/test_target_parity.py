"""Parity on the listings the headline is quoted on.

``tests/golden/listings/*.sass`` are the cubin frontend's renderings of the
shipped ``gemm_lrelu_f16`` (n = 1 184) and ``attn_fwd_f16`` targets, and
``tests/golden/targets.json.gz`` holds what the *reference* computed on them
(``make_target_golden.py``: ``anneal.py:123-213`` with ``SimulatorBackend``).

CPU tier: the committed listings are what the frontend renders from the built
cubins today (so the bench searches exactly these), the oracle reproduces the
reference byte for byte, and the reference's facts (classes, candidates,
cuts, simulate) are reproduced by the host frontend.
GPU tier: the device engine reproduces the reference histories byte for byte,
and agrees with the oracle on thousands of further chains (default and
``long`` schedules; the GEMM listing at the bench's own configuration).
"""
import hashlib

import numpy as np
import pytest

from conftest import oracle_many, target_golden
from golden_configs import CONFIGS
from oracle import oracle
from paper_2403_16863_b200 import AnnealConfig, parse_kernel, simulate
from paper_2403_16863_b200.machine import MachineConfig
from paper_2403_16863_b200.perturb import candidates
from paper_2403_16863_b200.tables import KernelTables

NAMES = ["gemm_lrelu_f16", "attn_fwd_f16"]
CUBINS = {"gemm_lrelu_f16": "gemm_lrelu.cubin", "attn_fwd_f16": "attn_fwd.cubin"}


def setup(name):
    rec = target_golden()["listings"][name]
    k = parse_kernel(rec["text"], name=name)
    return rec, k, KernelTables.build(k, MachineConfig())


@pytest.mark.parametrize("name", NAMES)
def test_committed_listing_is_the_shipped_cubin(name):
    """The bench decodes the shipped cubin; the goldens were made on this text."""
    from paper_2403_16863_b200.cubin import render_listing
    from paper_2403_16863_b200.targets import TARGET_DIR

    rec = target_golden()["listings"][name]
    got = render_listing((TARGET_DIR / CUBINS[name]).read_bytes(), name)
    assert got.text == rec["text"]
    assert got.n == rec["n"]


@pytest.mark.parametrize("name", NAMES)
def test_frontend_facts_match_reference(name):
    rec, k, t = setup(name)
    assert [ins.klass.value for ins in k.schedule] == rec["classes"]
    assert list(candidates(k).positions) == rec["cands"]
    assert list(k.block_boundaries) == rec["cuts"]
    assert rec["serialize_ok"]


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_reference(name):
    rec, k, t = setup(name)
    ol = oracle.OracleListing(t)
    assert ol.simulate(np.arange(t.n)) == rec["sim"]["total"]
    for w in rec["walks"]:
        assert ol.swap_legal(w["perm"]).tolist() == w["legal"]
    for cname, runs in rec["anneal"].items():
        cfg = AnnealConfig(**CONFIGS[cname])
        temps = cfg.temperatures()
        for seed, want in runs.items():
            hist, best, cur, summ = ol.anneal(int(seed), temps, unsafe=cfg.unsafe_moves)
            jsonl = oracle.history_jsonl(hist, summ["t0"], temps)
            assert jsonl == want["jsonl"], (cname, seed)
            assert best.tolist() == want["best"] and cur.tolist() == want["current"]
            assert summ["best_energy"] == want["best_energy"]


# ---------------------------------------------------------------- GPU tier
@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_device_legality_matches_reference_walks(name):
    from paper_2403_16863_b200.engine import get_context

    rec, k, t = setup(name)
    assert simulate(k).to_json() == rec["sim"]["json"]
    dk = get_context().kernel(t)
    n = t.n
    for w in rec["walks"]:
        los = np.arange(n - 1, dtype=np.int32)
        scheds = np.tile(np.asarray(w["perm"], dtype=np.uint16), (n - 1, 1))
        assert dk.legality(scheds, los).tolist() == w["legal"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_device_histories_byte_identical_to_reference(name):
    from paper_2403_16863_b200.anneal import anneal_batch_sim

    rec, k, t = setup(name)
    for cname, runs in rec["anneal"].items():
        cfg = AnnealConfig(**CONFIGS[cname])
        seeds = [int(s) for s in runs]
        states = anneal_batch_sim(k, MachineConfig(), cfg, seeds, tables=t)
        for seed, st in zip(seeds, states):
            want = runs[str(seed)]
            jsonl = st.history_jsonl()
            assert jsonl == want["jsonl"], (cname, seed)
            assert hashlib.sha256(jsonl.encode()).hexdigest() == want["sha256"]
            assert st.best_perm.tolist() == want["best"]
            assert st.current_perm.tolist() == want["current"]
            assert st.best_energy == want["best_energy"]
            assert st.ambiguous == 0


# chains per (listing, config): the GEMM default is the bench's own configuration
MANY = {("gemm_lrelu_f16", "default"): 4096, ("gemm_lrelu_f16", "long"): 512,
        ("attn_fwd_f16", "default"): 1024, ("attn_fwd_f16", "long"): 128}


@pytest.mark.gpu
@pytest.mark.parametrize("name,cname", sorted(MANY))
def test_device_chains_vs_oracle_on_target_listing(name, cname):
    """Thousands of seeds beyond the goldens, in one launch of the fused kernel (the
    bench's code path: lazy checkpoint offsets, speculative writes, ck_restore)."""
    from paper_2403_16863_b200.engine import get_context

    rec, k, t = setup(name)
    dk = get_context().kernel(t)
    cfg = AnnealConfig(**CONFIGS[cname])
    temps = cfg.temperatures()
    seeds = np.arange(50_000, 50_000 + MANY[(name, cname)], dtype=np.int64)
    hist, best, cur, summ = dk.anneal(seeds, temps)
    ref = oracle_many(oracle.OracleListing(t), seeds, temps)
    rejected = 0
    for c, (oh, ob, oc, os_) in enumerate(ref):
        assert np.array_equal(hist[c], oh), (name, cname, int(seeds[c]))
        assert np.array_equal(best[c], ob) and np.array_equal(cur[c], oc), int(seeds[c])
        assert summ["best_energy"][c] == os_["best_energy"]
        rejected += int((oh["status"] == 1).sum())
    assert int(summ["ambiguous"].sum()) == 0
    # the rejection path (ck_restore) is exercised, not just accepted moves
    assert rejected > 0 or cname == "default"


@pytest.mark.parametrize("name", NAMES)
def test_oracle_on_reference_facts_reproduces_reference(name):
    """The reference arm's path (bench.py --impl reference): oracle tables packed from the
    reference's own per-instruction facts, no product host code."""
    from oracle.golden_tables import tables_from_facts

    rec = target_golden()["listings"][name]
    ol = oracle.OracleListing(tables_from_facts(rec))
    assert ol.simulate(np.arange(rec["n"])) == rec["sim"]["total"]
    for cname in ("default", "long"):
        cfg = AnnealConfig(**CONFIGS[cname])
        temps = cfg.temperatures()
        for seed, want in rec["anneal"][cname].items():
            hist, best, cur, summ = ol.anneal(int(seed), temps)
            assert oracle.history_jsonl(hist, summ["t0"], temps) == want["jsonl"], (cname, seed)


@pytest.mark.parametrize("name", NAMES)
def test_product_tables_match_reference_facts(name):
    """The product's host table builder (tables.py) against the reference's facts."""
    from oracle.golden_tables import tables_from_facts

    rec, k, t = setup(name)
    g = tables_from_facts(rec)
    mask = np.uint32(0x00FFFFFF & ~(0xF << 17))  # scoreboard, class bits; no reuse/hw-only bits
    assert np.array_equal(t.ctrl & mask, g.ctrl & mask)
    assert np.array_equal(t.lat, g.lat) and np.array_equal(t.cut, g.cut)
    assert np.array_equal(t.nrefs, g.nrefs)

    def names(tab, i, which, order):
        row = getattr(tab, which).reshape(tab.n, tab.words)[i]
        return {order[b] for b in range(len(order)) if (int(row[b >> 6]) >> (b & 63)) & 1}

    gnames = {}
    for r, w in rec["rw"]:
        for x in sorted(set(r) | set(w)):
            gnames.setdefault(x, len(gnames))
    gorder = sorted(gnames, key=gnames.get)
    for i in range(t.n):
        for which in ("reads", "writes"):
            assert names(t, i, which, t.names) == names(g, i, which, gorder), (i, which)


# the sm_100 extension classes: no reference counterpart, so the device is
# pinned to the oracle on the extended tables (movable compute, exact packed-pair footprints,
# every non-movable instruction a fence) -- the engine at realistic candidate counts
EXT_MANY = {"gemm_lrelu_f16": 1024, "attn_fwd_f16": 256}


@pytest.mark.gpu
@pytest.mark.parametrize("classes", ["extended", "sm100"])
@pytest.mark.parametrize("name", sorted(EXT_MANY))
def test_device_chains_vs_oracle_extended_classes(name, classes):
    """The sm100 tables too (waiting compute, the uniform datapath and bulk copies movable;
    the guard rows only matter under hw_safe, which the oracle, like the reference, lacks)."""
    from paper_2403_16863_b200.engine import get_context

    rec, k, _ = setup(name)
    t = KernelTables.build(k, MachineConfig(), classes=classes)
    assert len(t.global_ids) > 300  # hundreds of candidates, not the reference's five
    dk = get_context().kernel(t)
    temps = AnnealConfig().temperatures()
    seeds = np.arange(70_000, 70_000 + EXT_MANY[name], dtype=np.int64)
    hist, best, cur, summ = dk.anneal(seeds, temps)
    ref = oracle_many(oracle.OracleListing(t), seeds, temps)
    priced = 0
    for c, (oh, ob, oc, os_) in enumerate(ref):
        assert np.array_equal(hist[c], oh), (name, int(seeds[c]))
        assert np.array_equal(best[c], ob) and np.array_equal(cur[c], oc), int(seeds[c])
        assert summ["best_energy"][c] == os_["best_energy"]
        priced += int((oh["status"] <= 1).sum())
    assert priced > 0 and int(summ["ambiguous"].sum()) == 0
