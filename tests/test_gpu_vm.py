"""GENERIC stage programs on the device VM (csrc/tm_vm.cu) against the
reference's generic interpreter (tests/golden/vm.npz, make_golden.py vm):
trigger counts, members attribution and instance lists for the shipped
custom patterns and grammar-coverage programs, on the hand graphs, 40
acceptance-corpus graphs x 3 deltas and a self-loop / timestamp-tie graph."""

from __future__ import annotations

import dataclasses
import json

import numpy as np
import pytest

from conftest import load_npz
from paper_2604_12241_b200 import plan as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tmb():
    import paper_2604_12241_b200 as tmb
    from paper_2604_12241_b200 import _lib
    _lib.load()
    return tmb


@pytest.fixture(scope="module")
def fx():
    z = load_npz("vm.npz")
    return z, json.loads(str(z["meta"])), [P.plan_from_dict(d) for d in json.loads(str(z["plans"]))]


def _graph(tmb, z, k, meta):
    e = z[f"edges{k}"]
    return tmb.DeviceGraph(e[:, 0], e[:, 1], e[:, 2], edge_amount=z[f"amount{k}"],
                           edge_currency=z[f"currency{k}"], currency_vocab=meta[k]["vocab"])


def _with_delta(plans, d, attribution="trigger"):
    return [dataclasses.replace(p, delta=d, attribution=attribution) for p in plans]


def test_vm_counts(tmb, fx):
    from paper_2604_12241_b200.vm import lower_program, vm_mine
    z, meta, plans = fx
    for k, m in enumerate(meta):
        g = _graph(tmb, z, k, meta)
        want = z[f"counts{k}"]
        for j, p in enumerate(_with_delta(plans, m["delta"])):
            got = vm_mine(g, lower_program(p, g.currency_vocab))
            np.testing.assert_array_equal(got, want[:, j], err_msg=f"{m['name']} d={m['delta']} {p.name}")
        g.free()


def test_vm_members(tmb, fx):
    from paper_2604_12241_b200.vm import lower_program, vm_members
    z, meta, plans = fx
    for k, m in enumerate(meta):
        g = _graph(tmb, z, k, meta)
        want = z[f"members{k}"]
        for j, p in enumerate(_with_delta(plans, m["delta"], "members")):
            got = vm_members(g, lower_program(p, g.currency_vocab))
            np.testing.assert_array_equal(got, want[:, j], err_msg=f"{m['name']} d={m['delta']} {p.name}")
        g.free()


def test_vm_instances(tmb, fx):
    from paper_2604_12241_b200.engine import decode_instances
    from paper_2604_12241_b200.vm import lower_program, vm_instance_stream
    z, meta, plans = fx
    names = [p.name for p in plans]
    idx = {n: i for i, n in enumerate(names)}
    n_checked = 0
    for k, m in enumerate(meta):
        want = z[f"rec{k}"].astype(np.int64)
        if len(want) == 0:
            continue
        g = _graph(tmb, z, k, meta)
        recs = []
        for j, p in enumerate(_with_delta(plans, m["delta"])):
            recs += decode_instances(vm_instance_stream(g, lower_program(p, g.currency_vocab), j, 0, g.edge_count),
                                     names)
        g.free()
        recs.sort(key=lambda r: (r.pattern, r.trigger_edge, r.member_edges))
        got = []
        for r in recs:
            got += [idx[r.pattern], r.trigger_edge, len(r.member_edges), len(r.member_nodes)]
            got += list(r.member_edges) + list(r.member_nodes)
        assert np.array_equal(np.array(got, dtype=np.int64), want), f"{m['name']} d={m['delta']}"
        n_checked += 1
    assert n_checked > 40


def test_mine_routes_generic_plans_to_the_vm(tmb, fx):
    """mine() with reference-compiled custom plans: same FeatureMatrix as the
    reference, hinted-family and VM columns mixed in one call."""
    z, meta, plans = fx
    k = next(i for i, m in enumerate(meta) if m["name"] == "corpus0")
    g = _graph(tmb, z, k, meta)
    ps = _with_delta(plans, meta[k]["delta"]) + [tmb.builtin_plan("sg_count", meta[k]["delta"])]
    fm = tmb.mine(g, ps)
    want = z[f"counts{k}"]
    for j, p in enumerate(plans):
        np.testing.assert_array_equal(fm.column(p.name), want[:, j], err_msg=p.name)
    fm2, inst = tmb.mine(g, ps, collect_instances=True)
    np.testing.assert_array_equal(fm2.values, fm.values)
    assert len(inst) > 0
    g.free()


def test_vm_predicates_exact_beyond_2p53(tmb):
    """Edge times near 2^60 against float amounts: the reference compares a
    Python int with a float exactly (engine.py:212-223); a double compare
    would disagree on 124 of the 400 edges (tests/golden/vm_bigtime.json,
    make_golden.py vm_bigtime)."""
    from conftest import GOLDEN
    from paper_2604_12241_b200.vm import lower_program, vm_mine
    fx = json.loads((GOLDEN / "vm_bigtime.json").read_text())
    e = np.asarray(fx["edges"], dtype=np.int64)
    g = tmb.DeviceGraph(e[:, 0], e[:, 1], e[:, 2], edge_amount=np.asarray(fx["amount"]),
                        edge_currency=np.zeros(len(e), dtype=np.int64), currency_vocab=["USD"])
    for case in fx["cases"]:
        for p, want in zip(case["plans"], case["counts"]):
            got = vm_mine(g, lower_program(P.plan_from_dict(p), g.currency_vocab))
            np.testing.assert_array_equal(got, np.asarray(want), err_msg=f"{p['name']} d={case['delta']}")
    g.free()
