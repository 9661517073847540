"""Pin the CPU oracle (oracle/tm_oracle.c) to the reference's own outputs.

Every expected value comes from tests/golden/*, produced by running the
reference (`tempmine.engine.mine`) — see tests/golden/make_golden.py.  The
oracle is then trusted as the checker of the GPU path on inputs for which no
reference output was recorded.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN, columns_of, corpus_graphs, load_hand, load_npz
from oracle.oracle import OracleGraph, column


def _cols(cols, delta):
    return [column(c["base"], delta, c["min_size"]) for c in cols]


def test_hand_cases():
    doc = load_hand()
    for case in doc["cases"]:
        e = np.array(case["edges"], dtype=np.int64)
        g = OracleGraph(e[:, 0], e[:, 1], e[:, 2])
        got = g.mine(_cols(doc["columns"], case["delta"]))
        np.testing.assert_array_equal(got, np.array(case["values"]), err_msg=f"{case['name']} d={case['delta']}")


@pytest.mark.skipif(not (GOLDEN / "corpus.npz").exists(), reason="corpus fixture not generated")
def test_acceptance_corpus():
    z = load_npz("corpus.npz")
    cols = columns_of(z)
    n = 0
    for i, edges, deltas, vals in corpus_graphs():
        g = OracleGraph(edges[:, 0], edges[:, 1], edges[:, 2])
        for k, d in enumerate(deltas.tolist()):
            got = g.mine(_cols(cols, d), threads=1)
            np.testing.assert_array_equal(got, vals[:, k, :], err_msg=f"graph {i} delta {d}")
            n += 1
    assert n == 600


@pytest.mark.skipif(not (GOLDEN / "ties.npz").exists(), reason="ties fixture not generated")
def test_ties_and_selfloops():
    import json
    z = load_npz("ties.npz")
    cols = columns_of(z)
    meta = json.loads(str(z["meta"]))
    for idx, m in enumerate(meta):
        g = OracleGraph(z[f"src{idx}"], z[f"dst{idx}"], z[f"time{idx}"])
        vals = z[f"values{idx}"]
        for k, d in enumerate(m["deltas"]):
            got = g.mine(_cols(cols, d))
            np.testing.assert_array_equal(got, vals[:, k, :], err_msg=f"ties {idx} delta {d}")


@pytest.mark.skipif(not (GOLDEN / "cfg1.npz").exists(), reason="cfg1 fixture not generated")
def test_cfg1_full_columns():
    from paper_2604_12241_b200 import synth
    z = load_npz("cfg1.npz")
    g0 = synth.generate(synth.CONFIGS["cfg1"])
    g = OracleGraph(g0.src, g0.dst, g0.time)
    got = g.mine(_cols(columns_of(z), 86400))
    np.testing.assert_array_equal(got, z["values"])


def test_csr_matches_lexsort(hand_doc):
    """Oracle adjacency == np.lexsort((eid, time, owner)) (txgraph.py:134-144)."""
    rng = np.random.default_rng(5)
    src = rng.integers(0, 30, 500)
    dst = rng.integers(0, 30, 500)
    t = rng.integers(0, 20, 500)
    g = OracleGraph(src, dst, t, node_count=31)
    eids = np.arange(500)
    for direction, owner, other in (("out", src, dst), ("in", dst, src)):
        indptr, nbr, tim, eid = g.export(direction)
        order = np.lexsort((eids, t, owner))
        np.testing.assert_array_equal(eid, order)
        np.testing.assert_array_equal(nbr, other[order])
        np.testing.assert_array_equal(tim, t[order])
        np.testing.assert_array_equal(indptr, np.concatenate([[0], np.cumsum(np.bincount(owner, minlength=31))]))


def test_thread_count_invariance():
    rng = np.random.default_rng(9)
    src = rng.integers(0, 200, 5000)
    dst = rng.integers(0, 200, 5000)
    t = rng.integers(0, 300, 5000)
    g = OracleGraph(src, dst, t)
    cols = [column(b, 40) for b in ("fan_in", "cycle_4", "cycle_6", "sg_count", "gs_count", "stack_count")]
    a = g.mine(cols, threads=1)
    b = g.mine(cols, threads=8)
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(g.mine(cols, 1000, 2000, threads=3), a[1000:2000])
