"""Per-rank compute of an N-GPU step, emulated on ONE B200 (only one GPU is
available to this build): for each rank r of world N, the device time of
exactly what rank r runs in `bench.py --gpus N` / `mine_distributed` —
tm_mine_prepare of its contiguous trigger range (its time slabs only) plus
its pieces — timed with CUDA events, rank after rank on the same GPU.
max over ranks = the N-GPU step's compute time without the all-gather.

    python tools/emulate_ranks.py [hi-large] [--worlds 1,2,4,8] [--pieces 4]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_12241_b200 as tmb  # noqa: E402
from paper_2604_12241_b200 import synth  # noqa: E402
from paper_2604_12241_b200.distributed import piece_bounds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="hi-large")
ap.add_argument("--worlds", default="1,2,4,8")
ap.add_argument("--pieces", type=int, default=4)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()

g0 = synth.time_ordered(synth.generate(synth.CONFIGS[a.config]))
g = tmb.DeviceGraph(g0.src, g0.dst, g0.time, node_count=g0.node_count)
descs = [tmb.lower_plan(p) for p in tmb.full_pattern_set(86400)]
E, C = g.edge_count, len(descs)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for world in [int(x) for x in a.worlds.split(",")]:
    pieces = a.pieces if world > 1 else 1
    _, sub, bounds = piece_bounds(E, world, pieces)
    out = torch.empty((pieces, max(sub, 1), C), dtype=torch.int64, device="cuda")
    per_rank = []
    for r in range(world):
        best = None
        for rep in range(a.reps + 1):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            lo0, hi0 = bounds[r][0][0], bounds[r][-1][1]
            if world > 1:
                tmb.prepare_views(g, descs, lo0, hi0, st.cuda_stream)
            for p, (lo, hi) in enumerate(bounds[r]):
                if hi > lo:
                    tmb.mine_rows_device(g, descs, lo, hi, out[p].data_ptr(), st.cuda_stream)
            if world > 1:
                tmb.release_views(g)
            e1.record(st)
            e1.synchronize()
            if rep and (best is None or e0.elapsed_time(e1) < best):
                best = e0.elapsed_time(e1)
        per_rank.append(best)
    mx = float(np.max(per_rank))
    print(json.dumps({"config": a.config, "world": world, "pieces": pieces, "rank_ms": per_rank,
                      "max_rank_ms": mx, "mean_rank_ms": float(np.mean(per_rank)),
                      "edges_per_s_compute": E / (mx / 1e3),
                      "note": "emulated on one GPU: per-rank prepare + pieces, all-gather excluded"}), flush=True)
g.free()
