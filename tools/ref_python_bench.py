"""The reference's own Python mining path on the GPU box's host cores, beside
the GPU, on sampled trigger blocks of a benchmark workload (test
infrastructure: oracle/ref_python.py; run `sh oracle/stage_ref.sh` in the
build container first so oracle/_ref/ travels with the snapshot).

    python tools/ref_python_bench.py [hi-large] [--blocks 64] [--block 1000]

1. the GPU mines all E triggers (device-resident graph, full pattern set);
2. the reference (`tempmine.engine._mine_range`, engine.py:607-646, on its
   own TemporalGraph and compiled plans) mines random contiguous 1000-trigger
   blocks with a fork pool of os.cpu_count() workers (engine.py:677-690);
3. prints one JSON line: the reference's edges/s on those blocks (wall time
   over P workers, EXTRAPOLATED to the full run), the CPU model and P, and
   the row-for-row comparison of the GPU output with the reference's rows.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="hi-large")
ap.add_argument("--blocks", type=int, default=64)
ap.add_argument("--block", type=int, default=1000)
ap.add_argument("--seed", type=int, default=77)
a = ap.parse_args()

from oracle import ref_python  # noqa: E402

if not ref_python.available():
    print(json.dumps({"config": a.config, "unavailable": "oracle/_ref/tempmine not staged (oracle/stage_ref.sh)"}))
    sys.exit(0)

import torch  # noqa: E402

import paper_2604_12241_b200 as tmb  # noqa: E402
from paper_2604_12241_b200 import synth  # noqa: E402

DELTA = 86400
t0 = time.perf_counter()
g0 = synth.time_ordered(synth.generate(synth.CONFIGS[a.config]))
E = g0.edge_count
gen_s = time.perf_counter() - t0
names = list(tmb.FULL_PATTERN_SET)

# GPU: every trigger, device output; only the sampled rows come back
g = tmb.DeviceGraph(g0.src, g0.dst, g0.time, node_count=g0.node_count)
descs = [tmb.lower_plan(p) for p in tmb.full_pattern_set(DELTA)]
out = torch.empty((E, len(descs)), dtype=torch.int64, device="cuda")
st = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
tmb.mine_rows_device(g, descs, 0, E, out.data_ptr(), st.cuda_stream)  # warm-up
e0.record(st)
tmb.mine_rows_device(g, descs, 0, E, out.data_ptr(), st.cuda_stream)
e1.record(st)
e1.synchronize()
gpu_ms = e0.elapsed_time(e1)

rng = np.random.default_rng(a.seed)
blocks = []
for _ in range(a.blocks):
    lo = int(rng.integers(0, max(1, E - a.block)))
    blocks.append((lo, min(lo + a.block, E)))
idx = torch.from_numpy(np.concatenate([np.arange(lo, hi) for lo, hi in blocks])).cuda()
got = out.index_select(0, idx).cpu().numpy()
del out
g.free()

ref = ref_python.RefPython(g0.src, g0.dst, g0.time, g0.node_count, names, DELTA)
P = os.cpu_count() or 1
rows, cpu_s, wall = ref.mine(blocks, P)
want = np.concatenate(rows, axis=0)
diff = got != want
n_rows = int(want.shape[0])
cpu = "unknown"
try:
    for line in Path("/proc/cpuinfo").read_text().splitlines():
        if line.startswith("model name"):
            cpu = line.split(":", 1)[1].strip()
            break
except OSError:
    pass
rate = n_rows / wall
print(json.dumps({
    "config": a.config, "n_edges": E, "columns": names, "delta": DELTA,
    "reference": "tempmine.engine._mine_range (engine.py:607-646), unmodified, staged from /root/reference "
                 "(oracle/stage_ref.sh); builtins on their hinted batch kernels, cycle_5/6 and gs_count on "
                 "the generic interpreter (SURVEY Appendix B DSL)",
    "blocks": len(blocks), "block_triggers": a.block, "rows": n_rows,
    "workers": P, "cpu": cpu, "wall_s": wall, "cpu_s_summed": cpu_s,
    "edges_per_s": rate, "edges_per_s_note": "EXTRAPOLATED: sampled-block rows / wall time with P fork "
                                             "workers (the full run does not finish in minutes)",
    "full_run_extrapolated_s": E / rate,
    "reference_graph_build_s": ref.build_s, "generate_s": gen_s,
    "gpu_full_call_ms": gpu_ms, "gpu_edges_per_s": E / (gpu_ms / 1e3),
    "parity": {"rows": n_rows, "mismatching_rows": int(diff.any(axis=1).sum()),
               "bad_columns": [names[j] for j in np.nonzero(diff.any(axis=0))[0]],
               "checker": "the reference itself (GPU rows vs _mine_range rows, bit-exact int64)"},
}), flush=True)
sys.exit(1 if diff.any() else 0)
