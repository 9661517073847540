"""Multi-GPU mining: replicate the graph, split triggers, one all-gather.

SURVEY.md §8e: every column of a trigger row depends only on the immutable
graph and the trigger (engine.py:12-14), so the trigger range [0, E) is cut
into `world` equal contiguous chunks (equal sizes are what
ncclAllGather needs; the last chunk is zero-padded), each rank mines its
chunk against its own HBM replica of the graph, and one in-place
all_gather_into_tensor over NVLink / NVSwitch assembles the int64 (E, C)
feature block on every GPU — the replacement of the reference's fork pool
and host-side block merge (engine.py:677-699).  One process per GPU,
torch.distributed for the plumbing.

Members-attribution columns (engine.py:629-640) add into the rows of every
member edge, not only the trigger's: each rank accumulates its triggers'
contributions into a full (E, C) block and the blocks are summed with one
all-reduce — the reference's merge_features sum (engine.py:106-120).

Transport: counts are int64, but nearly every column of a real graph stays
far below 2^31.  `narrow=True` gathers each piece as int32 plus a one-byte
overflow flag per rank; a piece whose flag is set anywhere is gathered again
as int64, so the assembled block is bit-exact either way while the common
case moves half the bytes over NVLink (HI-Large, C = 14: 10.1 instead of
20.2 GB).
"""

from __future__ import annotations

from typing import Callable

import numpy as np

INT32_MAX = 2**31 - 1


def partition(n_edges: int, world: int) -> tuple[int, list[tuple[int, int]]]:
    """Equal contiguous chunks: (chunk, [(lo, hi) per rank])."""
    if world < 1:
        raise ValueError("world must be >= 1")
    chunk = (n_edges + world - 1) // world if n_edges else 0
    return chunk, [(min(r * chunk, n_edges), min((r + 1) * chunk, n_edges)) for r in range(world)]


def _all_gather(dst, src, group, async_op=False):
    """all_gather_into_tensor on NCCL; the list form on gloo (CPU tests)."""
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        return dist.all_gather_into_tensor(dst, src, group=group, async_op=async_op)
    parts = list(dst.split(src.shape[0]))
    return dist.all_gather(parts, src, group=group, async_op=async_op)


def gather_rows(local, n_edges: int, group=None):
    """All-gather equal (chunk, C) blocks into (n_edges, C) on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    chunk, c = local.shape
    full = torch.empty((chunk * world, c), dtype=local.dtype, device=local.device)
    _all_gather(full, local, group)
    return full[:n_edges]


def mine_sharded(n_edges: int, n_cols: int, rank: int, world: int,
                 mine_block: Callable[[int, int, object], None], device="cuda", group=None):
    """Generic driver: `mine_block(lo, hi, out)` fills out[(hi-lo), C] for this
    rank's chunk; returns the gathered (n_edges, C) tensor."""
    import torch
    chunk, bounds = partition(n_edges, world)
    lo, hi = bounds[rank]
    local = torch.zeros((chunk, n_cols), dtype=torch.int64, device=device)
    if hi > lo:
        mine_block(lo, hi, local)
    return gather_rows(local, n_edges, group)


def piece_bounds(n_edges: int, world: int, pieces: int) -> tuple[int, int, list[list[tuple[int, int]]]]:
    """Piece assignment for a pipelined gather.

    Rank r owns the contiguous trigger range [r*C, (r+1)*C), C = pieces*sub
    (time-contiguous when edge ids are in time order, so the rank builds
    only the time slabs its triggers read: tm_mine_prepare), cut into
    `pieces` sub-ranges of `sub` rows.  Gathering piece p brings every
    rank's p-th sub-range (P = world*sub rows, rank-major); it is written to
    rows r*C + p*sub of the result while the next piece is mined.  Returns
    (P, sub, bounds[rank][piece] = (lo, hi)), ranges clamped to n_edges."""
    if world < 1 or pieces < 1:
        raise ValueError("world and pieces must be >= 1")
    sub = (n_edges + world * pieces - 1) // (world * pieces) if n_edges else 0
    P = sub * world
    C = sub * pieces
    bounds = [[(min(r * C + p * sub, n_edges), min(r * C + (p + 1) * sub, n_edges)) for p in range(pieces)]
              for r in range(world)]
    return P, sub, bounds


def rank_range(n_edges: int, world: int, pieces: int, rank: int) -> tuple[int, int]:
    """The contiguous trigger range of `rank` under piece_bounds."""
    _, sub, b = piece_bounds(n_edges, world, pieces)
    return b[rank][0][0], b[rank][-1][1]


def mine_pipelined(n_edges: int, n_cols: int, rank: int, world: int,
                   mine_block: Callable[[int, int, object], None], pieces: int = 4, device="cuda", group=None,
                   narrow: bool = False, stats: dict | None = None,
                   prepare: Callable[[int, int], None] | None = None,
                   on_mined: Callable[[], None] | None = None):
    """Like mine_sharded, but the gather of each piece is issued (async) as
    soon as the piece is mined, so it overlaps the next piece's mining.

    prepare(lo, hi), if given, runs once for the rank's whole range before
    its pieces (the per-step window tables / slab views, tm_mine_prepare);
    on_mined(), if given, runs once every piece is enqueued (bench: the
    compute-only timing event).
    narrow=True: int32 transport with per-piece overflow flags (module doc);
    `stats` (if given) receives {"pieces_int64": n} — pieces that had to be
    re-gathered at full width."""
    import torch
    P, sub, bounds = piece_bounds(n_edges, world, pieces)
    full = torch.empty((world * pieces * sub, n_cols), dtype=torch.int64, device=device)
    # gathered pieces arrive rank-major: piece p of rank r -> rows r*C + p*sub
    dest = full.view(world, pieces, sub, n_cols)
    local = torch.zeros((pieces, sub, n_cols), dtype=torch.int64, device=device)
    works = []
    stage = torch.empty((pieces * P, n_cols), dtype=torch.int32 if narrow else torch.int64, device=device)
    if narrow:
        flags = torch.zeros((pieces, 1), dtype=torch.int32, device=device)
        flags_all = torch.empty((world, pieces), dtype=torch.int32, device=device)
        narrow_local = torch.empty((pieces, sub, n_cols), dtype=torch.int32, device=device)
    if prepare is not None:
        lo0, hi0 = bounds[rank][0][0], bounds[rank][-1][1]
        if hi0 > lo0:
            prepare(lo0, hi0)
    for p in range(pieces):
        lo, hi = bounds[rank][p]
        if hi > lo:
            mine_block(lo, hi, local[p])
        if narrow:
            # counts are >= 0: one max decides whether int32 holds the piece
            if sub > 0:
                flags[p, 0] = (local[p].max() > INT32_MAX).to(torch.int32)
            narrow_local[p].copy_(local[p])  # wraps on overflow; the flag redoes the piece
            works.append(_all_gather(stage[p * P:(p + 1) * P], narrow_local[p], group, async_op=True))
        else:
            works.append(_all_gather(stage[p * P:(p + 1) * P], local[p], group, async_op=True))
    if on_mined is not None:
        on_mined()
    for w in works:
        w.wait()
    bad = np.zeros(pieces, dtype=np.int64)
    if narrow:
        _all_gather(flags_all.view(-1), flags.view(-1), group)  # rank r -> row r
        bad = flags_all.amax(dim=0).cpu().numpy()
    for p in range(pieces):
        if bad[p]:  # int32 wrapped somewhere in this piece: gather it again at full width
            wide = torch.empty((P, n_cols), dtype=torch.int64, device=device)
            _all_gather(wide, local[p], group)
            dest[:, p].copy_(wide.view(world, sub, n_cols))
        else:  # reorder (and widen) into the final rows
            dest[:, p].copy_(stage[p * P:(p + 1) * P].view(world, sub, n_cols))
    if stats is not None:
        stats["pieces_int64"] = int(np.count_nonzero(bad))
    return full[:n_edges]


def sum_members(n_edges: int, n_cols: int, rank: int, world: int,
                mine_range: Callable[[int, int, object], None], device="cuda", group=None):
    """Members attribution across ranks: `mine_range(lo, hi, acc)` ADDS the
    contributions of triggers [lo, hi) into the full (n_edges, C) block acc;
    rank r takes chunk r of the trigger range and one all-reduce(SUM)
    combines the blocks (engine.py:106-120 merge by sum)."""
    import torch
    import torch.distributed as dist
    _, bounds = partition(n_edges, world)
    lo, hi = bounds[rank]
    acc = torch.zeros((n_edges, n_cols), dtype=torch.int64, device=device)
    if hi > lo:
        mine_range(lo, hi, acc)
    dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    return acc


def mine_distributed(graph, plans, *, group=None, pieces: int = 4, narrow: bool = True):
    """`mine` across the ranks of the default (NCCL) process group.

    Each rank builds its own device replica of `graph` on
    torch.cuda.current_device(); returns the FeatureMatrix on every rank.
    Trigger-attribution columns: pipelined all-gather (≤ 32 columns per
    launch, as `mine`); members-attribution columns: all-reduce of full
    blocks.  GENERIC stage-VM plans are not distributed (UnsupportedPlanError).
    """
    import torch
    import torch.distributed as dist

    from . import _lib
    from .engine import (FeatureMatrix, _chunks, lower_all, mine_members_device, mine_rows_device, prepare_views,
                         release_views)
    from .graph import as_device_graph

    plans, descs = lower_all(plans)
    dg = as_device_graph(graph, torch.cuda.current_device())
    side = torch.cuda.Stream()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    E = dg.edge_count

    def on_side(fn, out):
        # launch on a non-NULL stream (NULL selects the graph's own stream),
        # then order the collective on the current stream after it
        side.wait_stream(torch.cuda.current_stream())
        out.record_stream(side)
        fn(out.data_ptr(), side.cuda_stream)
        torch.cuda.current_stream().wait_stream(side)

    values = torch.empty((E, len(descs)), dtype=torch.int64, device="cuda")
    trig = [i for i, d in enumerate(descs) if not d.members]
    memb = [i for i, d in enumerate(descs) if d.members]
    for part in _chunks(trig, _lib.MAX_PLANS):
        dp = [descs[i] for i in part]
        full = mine_pipelined(E, len(part), rank, world,
                              lambda lo, hi, out, dp=dp: on_side(
                                  lambda ptr, st: mine_rows_device(dg, dp, lo, hi, ptr, st), out),
                              pieces=pieces, device="cuda", group=group, narrow=narrow,
                              prepare=lambda lo, hi, dp=dp: prepare_views(dg, dp, lo, hi, side.cuda_stream))
        release_views(dg)
        values[:, part] = full
    for part in _chunks(memb, _lib.MAX_PLANS):
        dp = [descs[i] for i in part]
        acc = sum_members(E, len(part), rank, world,
                          lambda lo, hi, out, dp=dp: on_side(
                              lambda ptr, st: mine_members_device(dg, dp, lo, hi, ptr, st), out),
                          device="cuda", group=group)
        values[:, part] = acc
    host = values.cpu().numpy()
    return FeatureMatrix(tuple(p.name for p in plans), host, graph.edge_src, graph.edge_dst,
                         graph.edge_time, getattr(graph, "edge_label", dg.edge_label), device_graph=dg)
