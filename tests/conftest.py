"""Shared test setup.

Markers: ``gpu`` tests need a B200 (they call the CUDA library through the C
ABI and compare against the oracle / golden fixtures); everything else runs on
the CPU.  The oracle (oracle/) is test infrastructure and is imported only here
and in tests.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
for _p in (str(ROOT), str(ROOT / "tests")):
    if _p not in sys.path:
        sys.path.insert(0, _p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden_small():
    return dict(np.load(GOLDEN / "small.npz"))


@pytest.fixture(scope="session")
def golden_bench():
    return dict(np.load(GOLDEN / "bench.npz"))


@pytest.fixture(scope="session")
def golden_acceptance():
    return dict(np.load(GOLDEN / "acceptance.npz"))


@pytest.fixture(scope="session")
def golden_streams():
    return json.loads((GOLDEN / "streams.json").read_text())


@pytest.fixture(scope="session")
def golden_analogs():
    return json.loads((GOLDEN / "analogs.json").read_text())


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as orc
    orc.build()
    return orc


@pytest.fixture(scope="session")
def bench_graphs():
    from paper_2601_14476_b200 import benchmarks
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = benchmarks.load(name)[0]
        return cache[name]
    return get


@pytest.fixture(scope="session")
def golden_full():
    """Per-trial digests of whole benchmark batches (make_fullbatch.py, oracle)."""
    return dict(np.load(GOLDEN / "fullbatch.npz"))
