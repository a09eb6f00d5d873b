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


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


@lru_cache(maxsize=1)
def golden() -> dict:
    with gzip.open(GOLDEN, "rt") as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def gold() -> dict:
    return golden()


def listing_names(pred=None) -> list:
    data = golden()["listings"]
    return sorted(n for n, rec in data.items() if pred is None or pred(rec))
