"""Per-column cost diagnostic on a bench workload (GPU box).

    python tools/diag_columns.py [hi-small]

Mines each column of the full pattern set alone through the host API with
kernel event profiling on; prints light/heavy kernel ms and heavy-queue
length per column.
"""

import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

import paper_2604_12241_b200 as tmb  # noqa: E402
from paper_2604_12241_b200 import _lib, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "hi-small"
g0 = synth.time_ordered(synth.generate(synth.CONFIGS[name]))
g = tmb.DeviceGraph(g0.src, g0.dst, g0.time, node_count=g0.node_count)
_lib.check(_lib.load().tm_set_profiling(g.handle, 1), "prof")
names = list(tmb.FULL_PATTERN_SET) + ["cycle_7", "cycle_8"]
for n in names + ["ALL14"]:
    if n == "ALL14":
        descs = [tmb.lower_plan(p) for p in tmb.full_pattern_set(86400)]
    else:
        descs = [tmb.lower_plan(tmb.builtin_plan(n, 86400))]
    for rep in range(2):
        t = time.perf_counter()
        out = tmb.mine_rows(g, descs, 0, g.edge_count)
        wall = (time.perf_counter() - t) * 1e3
    st = tmb.last_stats(g)
    print(f"{n:12s} light {st.light_ms:9.3f} ms  heavy {st.heavy_ms:9.3f} ms  heavy_n {st.heavy_triggers:8d}  "
          f"wall {wall:8.1f} ms  sum {int(out.sum())}", flush=True)
