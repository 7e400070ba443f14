"""Shared test configuration.

Markers:
  gpu  — needs a B200 (runs on the GPU box via ``pytest -m gpu``); everything
         else runs on the CPU build container (``pytest -m "not gpu"``).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA (sm_100a) device")


def f32_from_hex(h: str) -> float:
    return float(np.frombuffer(bytes.fromhex(h), dtype="<f4")[0])


@pytest.fixture(scope="session")
def search_cases():
    return json.loads((GOLDEN / "search_cases.json").read_text())


@pytest.fixture(scope="session")
def standard_cases():
    return json.loads((GOLDEN / "standard_cases.json").read_text())


def load_fixture_dir(name: str):
    """Graph + PQ + matrix + queries of one golden fixture (oracle readers)."""
    from oracle import search_port as sp
    d = GOLDEN / name
    g = sp.read_lgr1(d / "graph.bin")
    pq = sp.read_lpq1(d / "pq.bin")
    out = dict(dir=d, graph=g, pq=pq)
    for key in ("matrix", "queries", "qn"):
        p = d / f"{key}.npy"
        if p.exists():
            out[key] = np.load(p)
    if (d / "deleted.bin").exists():
        out["deleted"] = sp.read_ldl1(d / "deleted.bin", g.n)
    return out
