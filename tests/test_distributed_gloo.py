"""N > 1 host logic on CPU: world_size 2 over gloo.  Each rank mines its
equal chunk (here with the oracle standing in as the block miner — the GPU
block miner is covered by -m gpu tests) and the all-gather must reassemble
exactly the single-process matrix."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_12241_b200.distributed import (mine_pipelined, mine_sharded, partition, piece_bounds,
                                                sum_members)


def test_partition_equal_chunks():
    chunk, b = partition(10, 3)
    assert chunk == 4 and b == [(0, 4), (4, 8), (8, 10)]
    chunk, b = partition(2, 4)
    assert chunk == 1 and b == [(0, 1), (1, 2), (2, 2), (2, 2)]
    assert partition(0, 2) == (0, [(0, 0), (0, 0)])
    with pytest.raises(ValueError):
        partition(5, 0)


def test_piece_bounds_cover_rows_in_order():
    for n, world, pieces in ((1001, 2, 4), (10, 3, 2), (4, 2, 4), (0, 2, 3), (7, 4, 1)):
        P, sub, b = piece_bounds(n, world, pieces)
        assert P == sub * world
        rows = []
        for r in range(world):  # rank r owns a contiguous range, cut into its pieces in order
            for p in range(pieces):
                lo, hi = b[r][p]
                assert hi - lo <= sub
                assert lo == min(n, (r * pieces + p) * sub)  # piece p of rank r -> rows r*C + p*sub
                rows.extend(range(lo, hi))
        assert rows == list(range(n))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, src, dst, t, names, delta, q):
    try:
        _work(rank, world, port, src, dst, t, names, delta, q)
    except BaseException as exc:  # report instead of leaving the peer waiting
        import traceback
        q.put((rank, traceback.format_exc()))
        raise


def _work(rank, world, port, src, dst, t, names, delta, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import OracleGraph, column
    og = OracleGraph(src, dst, t)
    cols = [column(n, delta) for n in names]

    def block(lo, hi, out):
        out[: hi - lo] = torch.from_numpy(og.mine(cols, lo, hi, threads=2))

    full = mine_sharded(len(src), len(cols), rank, world, block, device="cpu")
    piped = mine_pipelined(len(src), len(cols), rank, world, block, pieces=3, device="cpu")
    assert torch.equal(full, piped)
    # int32 transport: exact, no piece needs the int64 re-gather
    st = {}
    narrow = mine_pipelined(len(src), len(cols), rank, world, block, pieces=3, device="cpu", narrow=True,
                            stats=st)
    assert torch.equal(full, narrow) and st["pieces_int64"] == 0

    # a block with counts beyond int32 in one rank's part of one piece only:
    # that piece is re-gathered at full width, the others stay narrow
    r1 = piece_bounds(len(src), world, 3)[2][1]  # rank 1's pieces
    target = r1[1] if r1[1][1] > r1[1][0] else r1[0]

    def big_block(lo, hi, out):
        block(lo, hi, out)
        if rank == 1 and (lo, hi) == target:
            out[: hi - lo, 0] += 3 * 2**31

    want_big = mine_pipelined(len(src), len(cols), rank, world, big_block, pieces=3, device="cpu")
    st = {}
    got_big = mine_pipelined(len(src), len(cols), rank, world, big_block, pieces=3, device="cpu", narrow=True,
                             stats=st)
    assert torch.equal(want_big, got_big)
    assert st["pieces_int64"] == 1

    # members-style accumulation: each rank adds its triggers' contributions
    # into every row; the all-reduce sum equals one process doing all ranges
    def add_range(lo, hi, acc):
        for e in range(lo, hi):
            acc[e, 0] += 1
            acc[(e * 7) % len(src), 1] += e
    acc = sum_members(len(src), 2, rank, world, add_range, device="cpu")
    ref = torch.zeros_like(acc)
    add_range(0, len(src), ref)
    assert torch.equal(acc, ref)
    q.put((rank, full.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_edges", [1001, 4])
def test_two_rank_gather_matches_single(n_edges):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from oracle.oracle import OracleGraph, column
    rng = np.random.default_rng(n_edges)
    src = rng.integers(0, 40, n_edges)
    dst = rng.integers(0, 40, n_edges)
    t = rng.integers(0, 500, n_edges)
    names = ["fan_in", "cycle_3", "sg_count", "stack_count"]
    want = OracleGraph(src, dst, t).mine([column(n, 60) for n in names])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, src, dst, t, names, 60, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(2):
        r, val = q.get(timeout=120)
        assert not isinstance(val, str), val
        got[r] = val
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        np.testing.assert_array_equal(got[r], want)
