"""Host-side logic on CPU: synthetic generator vs the reference generator,
FeatureMatrix CSV format, column ordering and error behaviour."""

from __future__ import annotations

import hashlib
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, load_npz
from paper_2604_12241_b200 import plan as P
from paper_2604_12241_b200 import synth
from paper_2604_12241_b200.engine import EngineInvariantError, FeatureMatrix, merge_features, order_plans

REF = Path("/root/reference/pkg/src")


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


@pytest.mark.skipif(not (GOLDEN / "cfg1.npz").exists(), reason="cfg1 fixture not generated")
def test_synth_cfg1_bit_identical_to_reference_generator():
    z = load_npz("cfg1.npz")
    g = synth.generate(synth.CONFIGS["cfg1"])
    assert g.edge_count == int(z["edge_count"])
    assert _sha(g.src) == str(z["sha_src"])
    assert _sha(g.dst) == str(z["sha_dst"])
    assert _sha(g.time) == str(z["sha_time"])
    np.testing.assert_array_equal(g.truth_triggers, z["truth_triggers"])
    g0 = synth.generate(synth.SynthConfig(10_000, 100_000, 16 * 86400, seed=7))
    assert _sha(g0.src) == str(z["unplanted_sha_src"])
    assert _sha(g0.time) == str(z["unplanted_sha_time"])


def test_time_ordered_is_a_stable_permutation():
    g = synth.generate(synth.SynthConfig(500, 5000, 100_000, seed=3, plants=(synth.PlantSpec("cycle_3", 5),)))
    h = synth.time_ordered(g)
    assert (np.diff(h.time) >= 0).all()
    order = np.argsort(g.time, kind="stable")
    np.testing.assert_array_equal(h.src, g.src[order])
    np.testing.assert_array_equal(h.time[h.truth_triggers], g.time[g.truth_triggers])


@pytest.mark.skipif(not REF.exists(), reason="reference not mounted")
def test_synth_matches_reference_generator_live():
    import sys
    sys.path.insert(0, str(REF))
    from tempmine import synth as rs
    cfg = rs.SynthConfig(800, 6000, 50_000, seed=13, powerlaw_exponent=1.3,
                         plants=(rs.PlantSpec("sg_count", 7), rs.PlantSpec("stack_count", 4),
                                 rs.PlantSpec("cycle_2", 3)))
    recs, truth = rs.generate(cfg)
    ours = synth.generate(synth.SynthConfig(800, 6000, 50_000, seed=13, powerlaw_exponent=1.3,
                                            plants=(synth.PlantSpec("sg_count", 7),
                                                    synth.PlantSpec("stack_count", 4),
                                                    synth.PlantSpec("cycle_2", 3))))
    np.testing.assert_array_equal(ours.src, [r.src for r in recs])
    np.testing.assert_array_equal(ours.dst, [r.dst for r in recs])
    np.testing.assert_array_equal(ours.time, [r.timestamp for r in recs])
    np.testing.assert_array_equal(ours.amount, [r.amount for r in recs])
    np.testing.assert_array_equal(ours.label, [int(r.label) for r in recs])
    np.testing.assert_array_equal(ours.truth_triggers, [t.trigger_edge for t in truth])


def _fm(values, label):
    n = len(values)
    return FeatureMatrix(("fan_in", "sg_count"), np.asarray(values, dtype=np.int64),
                         np.arange(n, dtype=np.int64), np.arange(n, dtype=np.int64) + 1,
                         np.arange(n, dtype=np.int64) * 10, np.asarray(label, dtype=np.int8))


def test_to_csv_format(tmp_path):
    fm = _fm([[1, 0], [2, 5], [0, 0]], [0, -1, 1])
    p = tmp_path / "f.csv"
    fm.to_csv(str(p))
    assert p.read_bytes() == (b"edge_id,src,dst,timestamp,label,fan_in,sg_count\n"
                              b"0,0,1,0,0,1,0\n1,1,2,10,,2,5\n2,2,3,20,1,0,0\n")


@pytest.mark.skipif(not REF.exists(), reason="reference not mounted")
def test_to_csv_byte_identical_to_reference(tmp_path):
    import sys
    sys.path.insert(0, str(REF))
    from tempmine.engine import FeatureMatrix as RefFM
    rng = np.random.default_rng(1)
    vals = rng.integers(0, 10**12, (70000, 2))
    lab = rng.integers(-1, 2, 70000)
    ours = _fm(vals, lab)
    ref = RefFM(ours.columns, ours.values, ours.edge_src, ours.edge_dst, ours.edge_time, ours.edge_label)
    ours.to_csv(str(tmp_path / "a.csv"))
    ref.to_csv(str(tmp_path / "b.csv"))
    assert (tmp_path / "a.csv").read_bytes() == (tmp_path / "b.csv").read_bytes()


def test_order_plans_and_duplicates():
    plans = [P.builtin_plan("gs_count"), P.builtin_plan("stack_count"), P.builtin_plan("cycle_5"),
             P.builtin_plan("fan_in")]
    assert [p.name for p in order_plans(plans)] == ["fan_in", "stack_count", "gs_count", "cycle_5"]
    with pytest.raises(EngineInvariantError):
        order_plans(plans + [P.builtin_plan("fan_in", 3)])


def test_merge_features():
    a, b = _fm([[1, 2]], [0]), _fm([[3, 4]], [0])
    assert merge_features([a, b]).values.tolist() == [[4, 6]]
    with pytest.raises(EngineInvariantError):
        merge_features([])


def test_instance_stream_decode_and_jsonl(tmp_path):
    """Host half of collect_instances: records -> InstanceRecord with member
    sets deduped + sorted (engine.py:641-645) and the CLI JSONL (cli.py:163-167)."""
    import json
    from paper_2604_12241_b200.engine import InstanceRecord, decode_instances, write_instances
    buf = np.array([1, 7, 4, 3, 7, 2, 7, 5, 9, 3, 9,
                    0, 2, 1, 2, 2, 0, 1], dtype=np.int32)
    recs = decode_instances(buf, ["fan_in", "sg_count"])
    assert recs == [InstanceRecord("sg_count", 7, (2, 5, 7), (3, 9)),
                    InstanceRecord("fan_in", 2, (2,), (0, 1))]
    with pytest.raises(Exception):
        decode_instances(buf[:-1], ["fan_in", "sg_count"])
    path = tmp_path / "inst.jsonl"
    write_instances(str(path), recs)
    lines = path.read_text().splitlines()
    assert json.loads(lines[0]) == {"pattern": "sg_count", "trigger_edge": 7,
                                    "member_edges": [2, 5, 7], "member_nodes": [3, 9]}
    assert lines[1] == '{"pattern":"fan_in","trigger_edge":2,"member_edges":[2],"member_nodes":[0,1]}'
