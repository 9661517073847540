"""GPU parity: libtempmine_b200.so (via the C ABI) against the reference's
recorded outputs (tests/golden) and against the pinned CPU oracle.

Bar: bit-exact int64 equality for every column of every row.
"""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN, columns_of, corpus_graphs, load_hand, load_npz
from oracle.oracle import OracleGraph, column

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["auto", "slabs"])
def view_mode(request, monkeypatch):
    """Every parity case twice: the library's own choice of graph view (the
    global CSR on these small graphs) and the time-slab view forced
    (TM_SLABS=1, tm_slab.cu: windows spanning slab boundaries, halos,
    single-slab horizons)."""
    if request.param == "slabs":
        monkeypatch.setenv("TM_SLABS", "1")
    return request.param


@pytest.fixture(scope="module")
def tmb():
    import paper_2604_12241_b200 as tmb
    from paper_2604_12241_b200 import _lib
    _lib.load()  # the in-tree .so; raises (no fallback) if it is missing
    return tmb


def _descs(tmb, cols, delta):
    return [tmb.lower_plan(tmb.builtin_plan(c["base"], delta, c["min_size"], column=c["column"]))
            for c in cols]


def _mine(tmb, src, dst, t, cols, delta, node_count=None):
    g = tmb.DeviceGraph(src, dst, t, node_count=node_count)
    out = tmb.mine_rows(g, _descs(tmb, cols, delta), 0, g.edge_count)
    g.free()
    return out


def _split(tmb, cols):
    # at most 32 columns per launch
    return [cols[i:i + 32] for i in range(0, len(cols), 32)]


def test_hand_cases(tmb):
    doc = load_hand()
    for case in doc["cases"]:
        e = np.array(case["edges"], dtype=np.int64)
        got = _mine(tmb, e[:, 0], e[:, 1], e[:, 2], doc["columns"], case["delta"])
        np.testing.assert_array_equal(got, np.array(case["values"]), err_msg=f"{case['name']} d={case['delta']}")


def test_acceptance_corpus(tmb):
    z = load_npz("corpus.npz")
    cols = columns_of(z)
    n = 0
    for i, edges, deltas, vals in corpus_graphs():
        g = tmb.DeviceGraph(edges[:, 0], edges[:, 1], edges[:, 2])
        for k, d in enumerate(deltas.tolist()):
            got = tmb.mine_rows(g, _descs(tmb, cols, d), 0, g.edge_count)
            np.testing.assert_array_equal(got, vals[:, k, :], err_msg=f"graph {i} delta {d}")
            n += 1
        g.free()
    assert n == 600


@pytest.mark.skipif(not (GOLDEN / "ties.npz").exists(), reason="fixture not generated")
def test_ties_and_selfloops(tmb):
    z = load_npz("ties.npz")
    cols = columns_of(z)
    meta = json.loads(str(z["meta"]))
    for idx, m in enumerate(meta):
        g = tmb.DeviceGraph(z[f"src{idx}"], z[f"dst{idx}"], z[f"time{idx}"])
        for k, d in enumerate(m["deltas"]):
            got = tmb.mine_rows(g, _descs(tmb, cols, d), 0, g.edge_count)
            np.testing.assert_array_equal(got, z[f"values{idx}"][:, k, :], err_msg=f"ties {idx} delta {d}")
        g.free()


@pytest.mark.skipif(not (GOLDEN / "cfg1.npz").exists(), reason="fixture not generated")
def test_cfg1_reference_output(tmb):
    """cfg1: 102K edges, alpha = 2.1 giant hub — exercises the
    heavy (warp) queue; every column equals the reference's."""
    from paper_2604_12241_b200 import synth
    z = load_npz("cfg1.npz")
    g0 = synth.generate(synth.CONFIGS["cfg1"])
    cols = columns_of(z)
    got = _mine(tmb, g0.src, g0.dst, g0.time, cols, 86400)
    np.testing.assert_array_equal(got, z["values"])


def test_csr_matches_reference_layout(tmb):
    rng = np.random.default_rng(3)
    n, e = 300, 20000
    src = rng.integers(0, n, e)
    dst = rng.integers(0, n, e)
    t = rng.integers(0, 50, e) * 1000 + 10**12  # ties + large absolute times
    g = tmb.DeviceGraph(src, dst, t, node_count=n + 5)
    eids = np.arange(e)
    for direction, owner, other in (("out", src, dst), ("in", dst, src)):
        indptr, nbr, tim, eid = g.export_csr(direction)
        order = np.lexsort((eids, t, owner))  # txgraph.py:135-136
        np.testing.assert_array_equal(eid, order)
        np.testing.assert_array_equal(nbr, other[order])
        np.testing.assert_array_equal(tim, t[order])
        np.testing.assert_array_equal(indptr, np.concatenate([[0], np.cumsum(np.bincount(owner, minlength=n + 5))]))
    info = g.info()
    assert info.n_ranks == len(np.unique(t))
    st = g.stats
    assert st.mean_out_degree == pytest.approx(e / (n + 5))


ALL = ["fan_in", "fan_out", "deg_in_src", "deg_out_src", "deg_in_dst", "deg_out_dst", "cycle_2",
       "cycle_3", "cycle_4", "cycle_5", "cycle_6", "cycle_7", "cycle_8", "sg_count", "gs_count",
       "stack_count"]


def _oracle_vs_gpu(tmb, src, dst, t, delta, names=ALL, ks=None, rows=None):
    og = OracleGraph(src, dst, t)
    ks = ks or [None] * len(names)
    want = og.mine([column(nm, delta, k) for nm, k in zip(names, ks)])
    g = tmb.DeviceGraph(src, dst, t)
    descs = [tmb.lower_plan(tmb.builtin_plan(nm, delta, k)) for nm, k in zip(names, ks)]
    got = tmb.mine_rows(g, descs, 0, g.edge_count)
    st = tmb.last_stats(g)
    g.free()
    for j, nm in enumerate(names):
        bad = np.flatnonzero(got[:, j] != want[:, j])
        assert len(bad) == 0, f"{nm}: {len(bad)} rows differ, e.g. row {bad[:5]} got {got[bad[:5], j]} want {want[bad[:5], j]}"
    return st


def test_powerlaw_hubs_vs_oracle(tmb):
    """alpha = 1.0 / 2.1 hubs, parallel edges, many heavy triggers."""
    from paper_2604_12241_b200 import synth
    for alpha, n, m in ((2.1, 3000, 60000), (1.0, 20000, 200000)):
        cfg = synth.SynthConfig(n, m, 8 * 86400, seed=11, powerlaw_exponent=alpha,
                                plants=(synth.PlantSpec("sg_count", 40), synth.PlantSpec("cycle_4", 40)))
        g0 = synth.generate(cfg)
        st = _oracle_vs_gpu(tmb, g0.src, g0.dst, g0.time, 86400)
        assert st.heavy_triggers > 0  # the warp path was exercised


def test_long_windows_pull_and_filters_vs_oracle(tmb):
    """Long windows over power-law hubs: the backward sets overflow their
    exact lists, so chain tasks run with the B2/B3 Bloom filters; hub v
    triggers take the pull-V path (gs from u's side, cycles via useful a1);
    sg/gs thresholds 2 and 3 exercise the probe-free hits."""
    from paper_2604_12241_b200 import synth
    cfg = synth.SynthConfig(2500, 50000, 8 * 86400, seed=23, powerlaw_exponent=1.0,
                            plants=(synth.PlantSpec("cycle_4", 20), synth.PlantSpec("sg_count", 20)))
    g0 = synth.generate(cfg)
    names = ["cycle_3", "cycle_4", "cycle_5", "cycle_6", "sg_count", "gs_count", "stack_count",
             "gs_count", "sg_count"]
    ks = [None, None, None, None, None, None, None, 3, 3]
    st = _oracle_vs_gpu(tmb, g0.src, g0.dst, g0.time, 3 * 86400, names=names, ks=ks)
    assert st.heavy_triggers > 0


def test_dense_small_graph_vs_oracle(tmb):
    """Dense windows: long cycle chains, large intersections, self-loops."""
    rng = np.random.default_rng(21)
    n, e = 60, 6000
    src = rng.integers(0, n, e)
    dst = rng.integers(0, n, e)
    t = rng.integers(0, 400, e)
    _oracle_vs_gpu(tmb, src, dst, t, 25)
    _oracle_vs_gpu(tmb, src, dst, t, 0)
    _oracle_vs_gpu(tmb, src, dst, t, 3, names=["sg_count", "gs_count", "cycle_4", "cycle_5", "stack_count"],
                   ks=[1, 3, 2, 2, 3])


def test_window_monotone_in_delta(tmb):
    """Property (test_acceptance.py:244-261): every count is non-decreasing in
    delta for the unthresholded columns."""
    from paper_2604_12241_b200 import synth
    g0 = synth.generate(synth.SynthConfig(5000, 80000, 30 * 86400, seed=3, powerlaw_exponent=1.2))
    g = tmb.DeviceGraph(g0.src, g0.dst, g0.time)
    names = ["fan_in", "fan_out", "deg_in_src", "deg_out_dst", "cycle_2", "cycle_3", "cycle_4", "stack_count"]
    prev = None
    for d in (0, 600, 3600, 86400, 7 * 86400):
        cur = tmb.mine_rows(g, [tmb.lower_plan(tmb.builtin_plan(nm, d, 1)) for nm in names], 0, g.edge_count)
        if prev is not None:
            assert (cur >= prev).all()
        prev = cur
    g.free()


def test_ranges_and_determinism(tmb):
    rng = np.random.default_rng(8)
    src = rng.integers(0, 500, 30000)
    dst = rng.integers(0, 500, 30000)
    t = rng.integers(0, 10000, 30000)
    g = tmb.DeviceGraph(src, dst, t)
    descs = [tmb.lower_plan(p) for p in tmb.full_pattern_set(300)]
    full = tmb.mine_rows(g, descs, 0, g.edge_count)
    again = tmb.mine_rows(g, descs, 0, g.edge_count)
    np.testing.assert_array_equal(full, again)
    np.testing.assert_array_equal(tmb.mine_rows(g, descs, 1234, 20000), full[1234:20000])
    assert tmb.mine_rows(g, descs, 5, 5).shape == (0, 14)
    g.free()


def test_mine_api_drop_in(tmb):
    """mine(graph, plans) with a TemporalGraph-like host object: FeatureMatrix,
    column order per order_plans (engine.py:596-604), errors as the reference."""
    from types import SimpleNamespace
    e = np.array([(0, 2, 1), (0, 3, 2), (0, 4, 3), (2, 1, 4), (3, 1, 5), (4, 1, 6)], dtype=np.int64)
    g = SimpleNamespace(node_count=5, edge_src=e[:, 0], edge_dst=e[:, 1], edge_time=e[:, 2],
                        edge_label=np.full(6, -1, np.int8))
    plans = [tmb.builtin_plan("gs_count", 10), tmb.builtin_plan("sg_count", 10), tmb.builtin_plan("fan_in", 10)]
    fm = tmb.mine(g, plans, workers=4)
    assert fm.columns == ("fan_in", "sg_count", "gs_count")
    assert fm.column("sg_count").tolist() == [0, 0, 0, 0, 1, 1]
    assert fm.values.dtype == np.int64
    with pytest.raises(ValueError):
        tmb.mine(g, plans, workers=0)
    with pytest.raises(tmb.EngineInvariantError):
        tmb.mine(g, plans + [tmb.builtin_plan("fan_in", 3)])
    fm2, inst = tmb.mine(g, plans, collect_instances=True)
    np.testing.assert_array_equal(fm2.values, fm.values)
    sg = [r for r in inst if r.pattern == "sg_count"]
    # as the reference prints them (tempmine.engine.mine, collect_instances=True)
    assert [(r.trigger_edge, r.member_edges, r.member_nodes) for r in sg] == [
        (4, (0, 1, 3, 4), (0, 1, 2, 3)), (5, (0, 1, 2, 3, 4, 5), (0, 1, 2, 3, 4))]


def test_bad_graphs_raise(tmb):
    with pytest.raises(ValueError):
        tmb.DeviceGraph([0, 5], [1, 1], [0, 0], node_count=3)  # id outside [0, n)
    g = tmb.DeviceGraph([0], [1], [7])
    assert tmb.mine_rows(g, [tmb.lower_plan(tmb.builtin_plan("deg_out_src", 5))], 0, 1).tolist() == [[1]]
    with pytest.raises(ValueError):
        tmb.mine_rows(g, [tmb.lower_plan(tmb.builtin_plan("fan_in", 5))], 0, 2)
    g.free()


def test_single_timestamp_and_extreme_times(tmb):
    src = np.array([0, 1, 2, 0, 1], dtype=np.int64)
    dst = np.array([1, 2, 0, 2, 0], dtype=np.int64)
    for t0 in (0, 2**62, -(2**40)):
        t = np.full(5, t0, dtype=np.int64)
        _oracle_vs_gpu(tmb, src, dst, t, 0)
        _oracle_vs_gpu(tmb, src, dst, t, 2**61)


# ---------------------------------------------------------------- members

def _mdescs(tmb, cols, delta):
    import dataclasses
    return [dataclasses.replace(d, members=True) for d in _descs(tmb, cols, delta)]


def test_members_hand_cases(tmb):
    doc = json.loads((GOLDEN / "hand_members.json").read_text())
    for case in doc["cases"]:
        e = np.array(case["edges"], dtype=np.int64)
        g = tmb.DeviceGraph(e[:, 0], e[:, 1], e[:, 2])
        got = tmb.mine_members(g, _mdescs(tmb, doc["columns"], case["delta"]))
        g.free()
        np.testing.assert_array_equal(got, np.array(case["values"]), err_msg=f"{case['name']} d={case['delta']}")


def test_members_corpus(tmb):
    zm = load_npz("corpus_members.npz")
    cols = columns_of(zm)
    vals_all = zm["values"].astype(np.int64)
    off = load_npz("corpus.npz")["offsets"]
    for i, edges, deltas, _ in corpus_graphs():
        g = tmb.DeviceGraph(edges[:, 0], edges[:, 1], edges[:, 2])
        for k, d in enumerate(deltas.tolist()):
            got = tmb.mine_members(g, _mdescs(tmb, cols, d))
            np.testing.assert_array_equal(got, vals_all[off[i]:off[i + 1], k, :], err_msg=f"graph {i} delta {d}")
        g.free()


def test_members_ties(tmb):
    z = load_npz("ties.npz")
    zm = load_npz("ties_members.npz")
    meta = json.loads(str(z["meta"]))
    cols = columns_of(zm)
    g = tmb.DeviceGraph(z["src0"], z["dst0"], z["time0"])
    for k, d in enumerate(meta[0]["deltas"]):
        got = tmb.mine_members(g, _mdescs(tmb, cols, d))
        np.testing.assert_array_equal(got, zm["values0"][:, k, :], err_msg=f"ties members delta {d}")
    g.free()


def test_mine_mixed_attribution(tmb):
    """mine() with trigger and members columns in one call (engine.py:693-699)."""
    import dataclasses
    from types import SimpleNamespace
    doc = json.loads((GOLDEN / "hand_members.json").read_text())
    trig = load_hand()
    case = next(c for c in doc["cases"] if c["name"] == "sg_planted" and c["delta"] == 10)
    tcase = next(c for c in trig["cases"] if c["name"] == "sg_planted" and c["delta"] == 10)
    e = np.array(case["edges"], dtype=np.int64)
    g = SimpleNamespace(node_count=5, edge_src=e[:, 0], edge_dst=e[:, 1], edge_time=e[:, 2],
                        edge_label=np.full(len(e), -1, np.int8))
    sg_m = dataclasses.replace(tmb.builtin_plan("sg_count", 10), name="sg_m", attribution="members")
    fm = tmb.mine(g, [sg_m, tmb.builtin_plan("sg_count", 10)])
    names = [c["column"] for c in doc["columns"]]
    j = names.index("sg_count")
    assert fm.column("sg_m").tolist() == [r[j] for r in case["values"]]
    assert fm.column("sg_count").tolist() == [r[j] for r in tcase["values"]]


# ---------------------------------------------------------------- CSV export

def test_csv_export_gpu_matches_host_writer(tmb, tmp_path):
    """GPU int->text (tm_csv_format) == the host writer, which is
    byte-identical to engine.py:73-103 (tests/test_host.py)."""
    import dataclasses
    from types import SimpleNamespace
    rng = np.random.default_rng(4)
    n, e = 700, 40000
    src = rng.integers(0, n, e)
    dst = rng.integers(0, n, e)
    t = rng.integers(0, 5000, e) + 10**9
    lab = rng.integers(-1, 2, e).astype(np.int8)
    g = SimpleNamespace(node_count=n, edge_src=src, edge_dst=dst, edge_time=t, edge_label=lab)
    fm = tmb.mine(g, tmb.full_pattern_set(300))
    assert fm.device_graph is not None
    fm.to_csv(str(tmp_path / "gpu.csv"))
    host = dataclasses.replace(fm, device_graph=None)
    host.to_csv(str(tmp_path / "host.csv"))
    assert (tmp_path / "gpu.csv").read_bytes() == (tmp_path / "host.csv").read_bytes()
    # negative values / unlabeled rows format like "%d" / ""
    fm2 = dataclasses.replace(fm, values=-fm.values, edge_label=np.full(e, -1, np.int8))
    fm2.to_csv(str(tmp_path / "gpu2.csv"))
    dataclasses.replace(fm2, device_graph=None).to_csv(str(tmp_path / "host2.csv"))
    assert (tmp_path / "gpu2.csv").read_bytes() == (tmp_path / "host2.csv").read_bytes()


def test_members_cfg1(tmb):
    """cfg1 (alpha = 2.1 giant hub) in members attribution: the reference's
    generic interpreter needed ~19 min on 8 workers for these 13 columns."""
    from paper_2604_12241_b200 import synth
    zm = load_npz("cfg1_members.npz")
    g0 = synth.generate(synth.CONFIGS["cfg1"])
    g = tmb.DeviceGraph(g0.src, g0.dst, g0.time)
    got = tmb.mine_members(g, _mdescs(tmb, columns_of(zm), 86400))
    g.free()
    np.testing.assert_array_equal(got, zm["values"])


def test_empty_and_tiny_graphs(tmb):
    """E = 0 and E = 1: shapes and values as the reference (mine over no
    triggers returns an (E, C) int64 block)."""
    from types import SimpleNamespace
    e0 = np.zeros(0, dtype=np.int64)
    g = SimpleNamespace(node_count=0, edge_src=e0, edge_dst=e0, edge_time=e0,
                        edge_label=np.zeros(0, np.int8))
    fm = tmb.mine(g, tmb.full_pattern_set(100))
    assert fm.values.shape == (0, 14) and fm.values.dtype == np.int64
    import dataclasses
    m = dataclasses.replace(tmb.builtin_plan("stack_count", 5), name="st_m", attribution="members")
    assert tmb.mine(g, [m]).values.shape == (0, 1)
    one = SimpleNamespace(node_count=2, edge_src=np.array([0]), edge_dst=np.array([1]),
                          edge_time=np.array([5]), edge_label=np.array([-1], np.int8))
    fm1 = tmb.mine(one, tmb.full_pattern_set(0) + [m])
    assert fm1.column("deg_out_src").tolist() == [1] and fm1.column("deg_in_dst").tolist() == [1]
    assert int(fm1.values.sum()) == 2


# ---------------------------------------------------------------- instance lists

def _encode(recs, col_index):
    out = []
    for r in recs:
        out += [col_index[r.pattern], r.trigger_edge, len(r.member_edges), len(r.member_nodes)]
        out += list(r.member_edges) + list(r.member_nodes)
    return np.array(out, dtype=np.int64)


def test_instances_vs_reference(tmb):
    """collect_instances records (engine.py:629-645, 710-711) against the
    reference's own InstanceRecord lists: hand graphs at every delta and the
    first acceptance-corpus graphs (tests/golden/instances.npz)."""
    from paper_2604_12241_b200.engine import collect_instance_records
    z = load_npz("instances.npz")
    meta = json.loads(str(z["meta"]))
    cols_by = {"all": json.loads(str(z["all_columns"])), "corpus": json.loads(str(z["corpus_columns"]))}
    total = 0
    for k, m in enumerate(meta):
        cols = cols_by[m["specs"]]
        e = z[f"edges{k}"].astype(np.int64)
        g = tmb.DeviceGraph(e[:, 0], e[:, 1], e[:, 2])
        recs = []
        for part in _split(tmb, cols):
            recs += collect_instance_records(g, _descs(tmb, part, m["delta"]), [c["column"] for c in part])
        g.free()
        recs.sort(key=lambda r: (r.pattern, r.trigger_edge, r.member_edges))
        got = _encode(recs, {c["column"]: i for i, c in enumerate(cols)})
        want = z[f"rec{k}"].astype(np.int64)
        assert got.shape == want.shape and np.array_equal(got, want), f"{m['name']} d={m['delta']}"
        total += len(recs)
    assert total > 1000


def test_host_output_pieces_match_device_output(tmb):
    """Pinned host output of >= 1 M rows is mined in 8 pieces whose D2H
    overlaps the next piece (tm_mine): same values as the device-output
    path, and sampled rows equal the oracle."""
    import torch
    from paper_2604_12241_b200 import synth
    cfg = synth.SynthConfig(60000, 1_200_000, 6 * 86400, seed=31, powerlaw_exponent=1.1,
                            plants=(synth.PlantSpec("cycle_4", 30), synth.PlantSpec("sg_count", 30)))
    g0 = synth.generate(cfg)
    g = tmb.DeviceGraph(g0.src, g0.dst, g0.time, node_count=g0.node_count)
    descs = [tmb.lower_plan(p) for p in tmb.full_pattern_set(86400)]
    E, C = g.edge_count, len(descs)
    assert E >= 1 << 20
    pinned = torch.empty((E, C), dtype=torch.int64).pin_memory().numpy()
    tmb.mine_rows(g, descs, 0, E, out=pinned)
    dev = torch.empty((E, C), dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    tmb.mine_rows_device(g, descs, 0, E, dev.data_ptr(), s.cuda_stream)
    s.synchronize()
    assert np.array_equal(pinned, dev.cpu().numpy())
    og = OracleGraph(g0.src, g0.dst, g0.time)
    names = list(tmb.FULL_PATTERN_SET)
    for lo in (0, E // 3, E - 700):
        want = og.mine([column(n, 86400) for n in names], lo, lo + 700)
        assert np.array_equal(pinned[lo:lo + 700], want), lo
