"""Shared fixtures.  GPU tests carry @pytest.mark.gpu and run only on a B200."""
from __future__ import annotations

import gzip
import json
import sys
from functools import lru_cache
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "reference.json.gz"
TARGET_GOLDEN = ROOT / "tests" / "golden" / "targets.json.gz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


@lru_cache(maxsize=1)
def golden() -> dict:
    with gzip.open(GOLDEN, "rt") as fh:
        return json.load(fh)


@lru_cache(maxsize=1)
def target_golden() -> dict:
    """Reference-run goldens for the decoded sm_100a target listings
    (tests/golden/make_target_golden.py)."""
    with gzip.open(TARGET_GOLDEN, "rt") as fh:
        return json.load(fh)


def oracle_many(ol, seeds, temps, unsafe: bool = False) -> list:
    """The oracle over many seeds on all host cores (ctypes releases the GIL; the oracle
    keeps no global state)."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(os.cpu_count() or 1) as ex:
        return list(ex.map(lambda s: ol.anneal(int(s), temps, unsafe=unsafe), seeds))


@pytest.fixture(scope="session")
def gold() -> dict:
    return golden()


def listing_names(pred=None) -> list:
    data = golden()["listings"]
    return sorted(n for n, rec in data.items() if pred is None or pred(rec))
