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
"""

from __future__ import annotations

from typing import Callable

import numpy as np


def partition(n_edges: int, world: int) -> tuple[int, list[tuple[int, int]]]:
    """Equal contiguous chunks: (chunk, [(lo, hi) per rank])."""
    if world < 1:
        raise ValueError("world must be >= 1")
    chunk = (n_edges + world - 1) // world if n_edges else 0
    return chunk, [(min(r * chunk, n_edges), min((r + 1) * chunk, n_edges)) for r in range(world)]


def gather_rows(local, n_edges: int, group=None):
    """All-gather equal (chunk, C) blocks into (n_edges, C) on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    chunk, c = local.shape
    full = torch.empty((chunk * world, c), dtype=local.dtype, device=local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(full, local, group=group)
    else:  # gloo (CPU tests): list form
        parts = list(full.split(chunk))
        dist.all_gather(parts, local, group=group)
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
    """Interleaved piece assignment for a pipelined gather.

    The trigger range is cut into `pieces` global pieces of P rows (P a
    multiple of `world`); rank r mines sub-range r of every piece.  The
    all-gather of piece p then lands exactly on global rows [p*P, (p+1)*P)
    in order, so each piece's gather can start while the next piece is
    mined — no reordering pass.  Returns (P, sub = P // world,
    bounds[rank][piece] = (lo, hi)), ranges clamped to n_edges."""
    if world < 1 or pieces < 1:
        raise ValueError("world and pieces must be >= 1")
    sub = (n_edges + world * pieces - 1) // (world * pieces) if n_edges else 0
    P = sub * world
    bounds = [[(min(p * P + r * sub, n_edges), min(p * P + (r + 1) * sub, n_edges)) for p in range(pieces)]
              for r in range(world)]
    return P, sub, bounds


def mine_pipelined(n_edges: int, n_cols: int, rank: int, world: int,
                   mine_block: Callable[[int, int, object], None], pieces: int = 4, device="cuda", group=None):
    """Like mine_sharded, but the gather of each piece is issued (async) as
    soon as the piece is mined, so it overlaps the next piece's mining."""
    import torch
    import torch.distributed as dist
    P, sub, bounds = piece_bounds(n_edges, world, pieces)
    full = torch.empty((pieces * P, n_cols), dtype=torch.int64, device=device)
    local = torch.zeros((pieces, sub, n_cols), dtype=torch.int64, device=device)
    nccl = dist.get_backend(group) == "nccl"
    works = []
    for p in range(pieces):
        lo, hi = bounds[rank][p]
        if hi > lo:
            mine_block(lo, hi, local[p])
        dst = full[p * P:(p + 1) * P]
        if nccl:
            works.append(dist.all_gather_into_tensor(dst, local[p], group=group, async_op=True))
        else:  # gloo (CPU tests): list form
            works.append(dist.all_gather(list(dst.split(sub)), local[p], group=group, async_op=True))
    for w in works:
        w.wait()
    return full[:n_edges]


def mine_distributed(graph, plans, *, group=None):
    """`mine` across the ranks of the default (NCCL) process group.

    Each rank builds its own device replica of `graph` on
    torch.cuda.current_device(); returns the FeatureMatrix on every rank.
    """
    import torch
    import torch.distributed as dist

    from .engine import FeatureMatrix, lower_all, mine_rows_device
    from .graph import as_device_graph

    plans, descs = lower_all(plans)
    dg = as_device_graph(graph, torch.cuda.current_device())
    side = torch.cuda.Stream()

    def block(lo, hi, out):
        # launch on a non-NULL stream (NULL selects the graph's own stream),
        # then order the all-gather on the current stream after it
        side.wait_stream(torch.cuda.current_stream())
        out.record_stream(side)
        mine_rows_device(dg, descs, lo, hi, out.data_ptr(), side.cuda_stream)
        torch.cuda.current_stream().wait_stream(side)

    full = mine_pipelined(dg.edge_count, len(descs), dist.get_rank(group), dist.get_world_size(group),
                          block, device="cuda", group=group)
    values = full.cpu().numpy()
    return FeatureMatrix(tuple(p.name for p in plans), values, graph.edge_src, graph.edge_dst,
                         graph.edge_time, getattr(graph, "edge_label", dg.edge_label))
