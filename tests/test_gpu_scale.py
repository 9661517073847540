"""Parity at benchmark scale: the GPU output on the
IBM-AML-shaped workloads against the CPU oracle (pinned to the reference,
tests/test_oracle_golden.py), plus the drop-in paths a user takes at scale:
mine() into pinned host memory and the NCCL multi-GPU driver at world 1.

* HI-Small shape, ALL 5.1 M rows x 14 columns compared (oracle on every
  host thread);
* HI-Medium shape, sampled 1000-trigger blocks (the reference's _mine_range
  seam, engine.py:607-646);
* the cycle-length x window sweep (BASELINE configs[4]) at the long windows
  (3 d, 7 d) for cycle_5..7 on sampled triggers of the HI-Medium graph.
"""

from __future__ import annotations

import os
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def tmb():
    import paper_2604_12241_b200 as tmb
    from paper_2604_12241_b200 import _lib
    _lib.load()
    return tmb


def _graph(name):
    from paper_2604_12241_b200 import synth
    return synth.time_ordered(synth.generate(synth.CONFIGS[name]))


@pytest.fixture(scope="module")
def hi_medium():
    return _graph("hi-medium")


@pytest.fixture
def slabs(request, monkeypatch):
    """TM_SLABS: "auto" = the library's choice (the global view on this
    shape), "1" = force the time-slab view (tm_slab.cu)."""
    if request.param != "auto":
        monkeypatch.setenv("TM_SLABS", request.param)
    return request.param


@pytest.mark.parametrize("slabs", ["auto", "1"], indirect=True)
def test_hi_small_full_array_parity(tmb, slabs):
    from oracle.oracle import OracleGraph, column
    g0 = _graph("hi-small")
    names = list(tmb.FULL_PATTERN_SET)
    g = tmb.DeviceGraph(g0.src, g0.dst, g0.time, node_count=g0.node_count)
    got = tmb.mine_rows(g, [tmb.lower_plan(p) for p in tmb.full_pattern_set(86400)], 0, g.edge_count)
    g.free()
    want = OracleGraph(g0.src, g0.dst, g0.time, node_count=g0.node_count).mine(
        [column(n, 86400) for n in names], threads=THREADS)
    assert got.shape == want.shape == (g0.edge_count, 14)
    bad = [n for j, n in enumerate(names) if not np.array_equal(got[:, j], want[:, j])]
    assert not bad, bad


def _blocks(E, n, size, seed):
    rng = np.random.default_rng(seed)
    for _ in range(n):
        lo = int(rng.integers(0, E - size))
        yield lo, lo + size


@pytest.mark.parametrize("slabs", ["auto", "1"], indirect=True)
def test_hi_medium_sampled_blocks(tmb, hi_medium, slabs):
    from oracle.oracle import OracleGraph, column
    g0 = hi_medium
    names = list(tmb.FULL_PATTERN_SET)
    g = tmb.DeviceGraph(g0.src, g0.dst, g0.time, node_count=g0.node_count)
    full = tmb.mine_rows(g, [tmb.lower_plan(p) for p in tmb.full_pattern_set(86400)], 0, g.edge_count)
    g.free()
    og = OracleGraph(g0.src, g0.dst, g0.time, node_count=g0.node_count)
    cols = [column(n, 86400) for n in names]
    for lo, hi in _blocks(g0.edge_count, 256, 1000, seed=5):
        want = og.mine(cols, lo, hi, threads=THREADS)
        np.testing.assert_array_equal(full[lo:hi], want, err_msg=f"block [{lo},{hi})")


@pytest.mark.parametrize("delta", [3 * 86400, 7 * 86400])
def test_sweep_long_windows_sampled(tmb, hi_medium, delta):
    """cycle_5..7 at long windows: chain enumeration over hubs with Bloom
    filters and pull tasks; triggers sampled (mined on their own ranges)."""
    from oracle.oracle import OracleGraph, column
    g0 = hi_medium
    names = ["cycle_5", "cycle_6", "cycle_7"] if delta <= 3 * 86400 else ["cycle_5", "cycle_6"]
    g = tmb.DeviceGraph(g0.src, g0.dst, g0.time, node_count=g0.node_count)
    og = OracleGraph(g0.src, g0.dst, g0.time, node_count=g0.node_count)
    descs = [tmb.lower_plan(tmb.builtin_plan(n, delta)) for n in names]
    cols = [column(n, delta) for n in names]
    t_end = time.time() + 240
    checked = 0
    for lo, hi in _blocks(g0.edge_count, 64, 20, seed=delta):
        got = tmb.mine_rows(g, descs, lo, hi)
        want = og.mine(cols, lo, hi, threads=THREADS)
        np.testing.assert_array_equal(got, want, err_msg=f"delta {delta} block [{lo},{hi})")
        checked += 1
        if time.time() > t_end:
            break
    g.free()
    assert checked >= 8


def test_mine_writes_pinned_values(tmb):
    """The drop-in mine() returns values in page-locked memory (overlapped
    D2H) that equal mine_rows; a second call re-uses the pinned pool."""
    from types import SimpleNamespace

    from paper_2604_12241_b200 import hostmem, synth
    g0 = synth.generate(synth.SynthConfig(20000, 400000, 8 * 86400, seed=4, powerlaw_exponent=1.0))
    hg = SimpleNamespace(node_count=g0.node_count, edge_src=g0.src, edge_dst=g0.dst, edge_time=g0.time,
                         edge_label=g0.label)
    plans = tmb.full_pattern_set(86400)
    fm = tmb.mine(hg, plans)
    assert hostmem.is_pinned(fm.values)
    dg = fm.device_graph
    want = tmb.mine_rows(dg, [tmb.lower_plan(p) for p in tmb.order_plans(plans)], 0, dg.edge_count)
    np.testing.assert_array_equal(fm.values, want)
    dg.free()
    del fm
    fm2 = tmb.mine(hg, plans)
    np.testing.assert_array_equal(fm2.values, want)
    fm2.device_graph.free()


def test_mine_distributed_nccl_world1(tmb):
    """The multi-GPU driver over NCCL at world size 1 (the only size a one-GPU
    box allows): pipelined pieces, int32 transport and the members
    all-reduce must reproduce mine() exactly."""
    import dataclasses
    import socket

    import torch
    import torch.distributed as dist

    from paper_2604_12241_b200 import synth
    from paper_2604_12241_b200.distributed import mine_distributed
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        g0 = synth.generate(synth.SynthConfig(5000, 100000, 8 * 86400, seed=9, powerlaw_exponent=1.0,
                                              plants=(synth.PlantSpec("sg_count", 30),)))
        from types import SimpleNamespace
        hg = SimpleNamespace(node_count=g0.node_count, edge_src=g0.src, edge_dst=g0.dst, edge_time=g0.time,
                             edge_label=g0.label)
        plans = tmb.full_pattern_set(86400)
        members = [dataclasses.replace(tmb.builtin_plan(n, 86400), name=f"{n}_m", attribution="members")
                   for n in ("cycle_3", "sg_count", "stack_count")]
        fm = mine_distributed(hg, plans + members, pieces=3, narrow=True)
        ref = tmb.mine(hg, plans + members)
        assert fm.columns == ref.columns
        np.testing.assert_array_equal(fm.values, ref.values)
        wide = mine_distributed(hg, plans, pieces=2, narrow=False)
        np.testing.assert_array_equal(wide.values, ref.values[:, :14])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("slabs", ["1"], indirect=True)
def test_prepared_rank_views_match_full_call(tmb, slabs):
    """tm_mine_prepare on one rank's contiguous, time-ordered trigger range
    builds only that range's time slabs; mining the rank's pieces against
    those views must equal one full call (HI-Small, 4 simulated ranks x 3
    pieces, the multi-GPU step's layout: distributed.piece_bounds)."""
    import torch

    from paper_2604_12241_b200.distributed import piece_bounds
    g0 = _graph("hi-small")
    g = tmb.DeviceGraph(g0.src, g0.dst, g0.time, node_count=g0.node_count)
    descs = [tmb.lower_plan(p) for p in tmb.full_pattern_set(86400)]
    E = g.edge_count
    want = torch.empty((E, len(descs)), dtype=torch.int64, device="cuda")
    tmb.mine_rows_device(g, descs, 0, E, want.data_ptr())
    got = torch.full((E, len(descs)), -1, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()  # the library mines on the graph's own stream
    world, pieces = 4, 3
    _, _, bounds = piece_bounds(E, world, pieces)
    for r in range(world):
        lo0, hi0 = bounds[r][0][0], bounds[r][-1][1]
        tmb.prepare_views(g, descs, lo0, hi0)
        for lo, hi in bounds[r]:
            if hi > lo:
                tmb.mine_rows_device(g, descs, lo, hi, got[lo:hi].data_ptr())
        tmb.release_views(g)
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    g.free()
