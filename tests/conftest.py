"""Shared fixtures.  `gpu` marks tests that need a B200 (run on the GPU box
with `pytest -m gpu`); everything else runs on CPU."""

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
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def load_hand():
    return json.loads((GOLDEN / "hand_cases.json").read_text())


def load_npz(name: str):
    return np.load(GOLDEN / name, allow_pickle=False)


def corpus_graphs():
    """Yields (index, edges[E,3], deltas[3], values[E,3,C]) of the C1 corpus."""
    z = load_npz("corpus.npz")
    edges, off, deltas, vals = z["edges"].astype(np.int64), z["offsets"], z["deltas"], z["values"]
    for i in range(len(off) - 1):
        a, b = off[i], off[i + 1]
        yield i, edges[a:b], deltas[i], vals[a:b].astype(np.int64)


def columns_of(z) -> list[dict]:
    return json.loads(str(z["columns"]))


@pytest.fixture(scope="session")
def hand_doc():
    return load_hand()
