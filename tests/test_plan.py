"""Drop-in lowering: the reference's compiled ExecutionPlans (recorded in
tests/golden/plans.json by the reference's compile_pattern) map onto the GPU
families exactly as _kernel_fn dispatches them (engine.py:569-589); GENERIC
plans of the extended families and force_generic builtins are recognized
structurally; everything else is rejected (no CPU fallback)."""

from __future__ import annotations

import json
from pathlib import Path

import pytest

from conftest import GOLDEN
from paper_2604_12241_b200 import plan as P
from paper_2604_12241_b200._lib import UnsupportedPlanError

# expected tm_plan_desc per base column: (family, endpoint, direction, exclude, cycle_len, default K)
EXPECTED = {
    "fan_in": (1, 1, 0, 1, 0, 1), "fan_out": (1, 0, 1, 1, 0, 1),
    "deg_in_src": (2, 0, 0, 0, 0, 1), "deg_out_src": (2, 0, 1, 0, 0, 1),
    "deg_in_dst": (2, 1, 0, 0, 0, 1), "deg_out_dst": (2, 1, 1, 0, 0, 1),
    "cycle_2": (3, 0, 0, 0, 2, 1), "cycle_3": (3, 0, 0, 0, 3, 1), "cycle_4": (3, 0, 0, 0, 4, 1),
    "cycle_5": (3, 0, 0, 0, 5, 1), "cycle_6": (3, 0, 0, 0, 6, 1), "cycle_7": (3, 0, 0, 0, 7, 1),
    "cycle_8": (3, 0, 0, 0, 8, 1), "sg_count": (4, 0, 0, 0, 0, 2), "gs_count": (5, 0, 0, 0, 0, 2),
    "stack_count": (6, 0, 0, 0, 0, 1),
}


def _obj(d):
    """Rebuild a reference ExecutionPlan (from dataclasses.asdict) as objects."""
    return P.plan_from_dict(d)


def _entries():
    return json.loads((GOLDEN / "plans.json").read_text())["plans"]


def _expect(base, k, delta):
    fam, ep, dr, ex, cl, k0 = EXPECTED[base]
    return P.PlanDesc(fam, ep, dr, ex, cl, k0 if k is None else k, delta)


def test_reference_plans_lower_to_expected_families():
    n = 0
    for e in _entries():
        if e["base"] is None:
            continue
        got = P.lower_plan(_obj(e["plan"]))
        assert got == _expect(e["base"], e["min_size"], e["plan"]["delta"]), (e["column"], e["force_generic"])
        n += 1
    assert n >= 50


def test_own_builders_match_reference_structure():
    seen = set()
    for e in _entries():
        if e["base"] is None or e["min_size"] is not None or e["force_generic"]:
            continue
        ref = _obj(e["plan"])
        ours = P.builtin_plan(e["base"], delta=ref.delta)
        assert P.canonical_shape(ours) == P.canonical_shape(ref), e["base"]
        assert ours.kernel_hint == ref.kernel_hint
        assert ours.emission.min_size == ref.emission.min_size
        seen.add(e["base"])
    assert seen == set(EXPECTED)


@pytest.mark.parametrize("name", ["spray_union", "filtered_senders", "sg_ordered", "stack_forward",
                                  "chain_5cycle"])
def test_unrecognized_custom_patterns_are_rejected(name):
    e = next(x for x in _entries() if x["column"] == name)
    with pytest.raises(UnsupportedPlanError):
        P.lower_plan(_obj(e["plan"]))


def test_members_attribution_lowering():
    import dataclasses
    p = dataclasses.replace(P.builtin_plan("sg_count"), attribution="members")
    d = P.lower_plan(p)
    assert d.members and d.family == 4 and d.min_size == 2
    assert not P.lower_plan(P.builtin_plan("sg_count")).members
    with pytest.raises(UnsupportedPlanError):
        P.lower_plan(dataclasses.replace(p, attribution="edges"))


def test_bad_parameters():
    import dataclasses
    p = P.builtin_plan("fan_in")
    with pytest.raises(ValueError):
        P.lower_plan(dataclasses.replace(p, delta=-1))
    with pytest.raises(ValueError):
        P.lower_plan(dataclasses.replace(p, emission=dataclasses.replace(p.emission, min_size=0)))


def test_full_pattern_set_is_c14():
    plans = P.full_pattern_set(86400)
    assert len(plans) == 14
    assert [p.name for p in plans][:11] == list(P.BUILTIN_COLUMNS)
    assert {P.lower_plan(p).delta for p in plans} == {86400}


@pytest.mark.skipif(not Path("/root/reference/pkg/src/tempmine").exists(), reason="reference not mounted")
def test_live_reference_compile_pattern():
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    from tempmine import plan as rplan
    from tempmine.txgraph import GraphStats
    stats = GraphStats(3.0, 3.0, 10.0, 10.0)
    for name in rplan.BUILTIN_COLUMNS:
        vp = rplan.load_builtin(name)
        for forced in (False, True):
            p = rplan.compile_pattern(vp, stats, force_generic=forced)
            assert P.lower_plan(p) == _expect(name, None, vp.delta)
