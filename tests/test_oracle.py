"""Pin the CPU oracle (oracle/sip_oracle.c) to the reference's own outputs.

Every annealing history the reference produced (tests/golden/make_golden.py)
must be reproduced byte for byte by the oracle before the oracle is trusted
as the checker of the CUDA path.
"""
import hashlib

import numpy as np
import pytest

from conftest import golden, listing_names
from oracle import oracle
from paper_2403_16863_b200 import AnnealConfig, parse_kernel
from paper_2403_16863_b200.machine import MachineConfig
from paper_2403_16863_b200.tables import KernelTables

from golden_configs import CONFIGS

ANNEAL_NAMES = listing_names(lambda r: "anneal" in r)
SIM_NAMES = listing_names(lambda r: "sim" in r)
WALK_NAMES = listing_names(lambda r: r["walks"])


def tables_for(name):
    rec = golden()["listings"][name]
    k = parse_kernel(rec["text"], name=name)
    return k, KernelTables.build(k, MachineConfig())


@pytest.mark.parametrize("name", SIM_NAMES)
def test_oracle_simulate(name):
    k, t = tables_for(name)
    assert oracle.OracleListing(t).simulate(np.arange(t.n)) == golden()["listings"][name]["sim"]["total"]


@pytest.mark.parametrize("name", WALK_NAMES)
def test_oracle_swap_legal_along_walks(name):
    k, t = tables_for(name)
    ol = oracle.OracleListing(t)
    for w in golden()["listings"][name]["walks"]:
        assert ol.swap_legal(w["perm"]).tolist() == w["legal"]


@pytest.mark.parametrize("name", ANNEAL_NAMES)
def test_oracle_anneal_histories(name):
    k, t = tables_for(name)
    ol = oracle.OracleListing(t)
    for cname, runs in golden()["listings"][name]["anneal"].items():
        cfg_kw = CONFIGS[cname]
        for seed, want in runs.items():
            cfg = AnnealConfig(seed=int(seed), **cfg_kw)
            temps = oracle.temperatures(cfg.t_max, cfg.cooling, cfg.iteration_budget)
            hist, best, cur, summ = ol.anneal(int(seed), temps, unsafe=cfg.unsafe_moves)
            jsonl = oracle.history_jsonl(hist, summ["t0"], temps)
            if "jsonl" in want:
                assert jsonl == want["jsonl"], (cname, seed)
            assert hashlib.sha256(jsonl.encode()).hexdigest() == want["sha256"], (cname, seed)
            assert best.tolist() == want["best"]
            assert cur.tolist() == want["current"]
            assert summ["best_energy"] == want["best_energy"]
            assert summ["t0"] == want["baseline"]


def test_oracle_sample_inputs():
    kinds = {"int8": 1, "int16": 2, "int32": 4}
    dists = {"uniform": 0, "small": 1, "zero": 2}
    for rec in golden()["samples"]:
        specs = [(5, kinds[rec["kind"]], dists[rec["dist"]]), (3, 4, 0)]
        b0, b1 = oracle.sample_inputs(rec["seed"], rec["index"], specs)
        assert b0.hex() == rec["buf0"] and b1.hex() == rec["buf1"], rec


def _edge():
    import json
    from pathlib import Path

    return json.loads((Path(__file__).parent / "golden" / "edge.json").read_text())


@pytest.mark.parametrize("name", sorted(_edge()))
def test_oracle_edge_listing_histories(name):
    """Boundaries, no legal move, cuts, all-candidate and tiny listings: the oracle
    reproduces the reference's histories (tests/golden/make_edge_golden.py)."""
    rec = _edge()[name]
    k = parse_kernel(rec["text"], name=name)
    ol = oracle.OracleListing(KernelTables.build(k, MachineConfig()))
    for cname, runs in rec["anneal"].items():
        cfg_kw = CONFIGS[cname]
        for seed, want in runs.items():
            cfg = AnnealConfig(seed=int(seed), **cfg_kw)
            temps = oracle.temperatures(cfg.t_max, cfg.cooling, cfg.iteration_budget)
            hist, best, cur, summ = ol.anneal(int(seed), temps, unsafe=cfg.unsafe_moves)
            jsonl = oracle.history_jsonl(hist, summ["t0"], temps)
            assert hashlib.sha256(jsonl.encode()).hexdigest() == want["sha256"], (cname, seed)
            assert best.tolist() == want["best"] and cur.tolist() == want["current"], (cname, seed)
