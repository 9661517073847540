"""End-to-end phase timing through the public API (GPU box):
python tools/diag_e2e.py [hi-small]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import os
if len(sys.argv) > 3:
    os.environ["TM_LIB"] = os.path.abspath(sys.argv[3])
import paper_2604_12241_b200 as tmb  # noqa: E402
from paper_2604_12241_b200 import synth  # noqa: E402

if os.environ.get("TM_BIND") == "1":  # pin the process to the GPU's NUMA-local cores
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
    cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
    cpus &= os.sched_getaffinity(0)
    if cpus:
        os.sched_setaffinity(0, cpus)
    print(f"bound to {len(cpus)} cpus: {sorted(cpus)[:4]}...", flush=True)
name = sys.argv[1] if len(sys.argv) > 1 else "hi-small"
g0 = synth.time_ordered(synth.generate(synth.CONFIGS[name]))
pin = lambda x: torch.from_numpy(np.ascontiguousarray(x, dtype=np.int64)).pin_memory().numpy()
hs, hd, ht = pin(g0.src), pin(g0.dst), pin(g0.time)
descs = [tmb.lower_plan(p) for p in tmb.full_pattern_set(86400)]
hout = torch.empty((g0.edge_count, len(descs)), dtype=torch.int64).pin_memory().numpy()
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    t0 = time.perf_counter()
    g = tmb.DeviceGraph(hs, hd, ht, node_count=g0.node_count)
    t1 = time.perf_counter()
    tmb.mine_rows(g, descs, 0, g.edge_count, out=hout)
    t2 = time.perf_counter()
    g.free()
    t3 = time.perf_counter()
    print(f"rep {rep}: build {1e3*(t1-t0):7.2f} ms  mine+D2H {1e3*(t2-t1):7.2f} ms  free {1e3*(t3-t2):6.2f} ms  "
          f"total {1e3*(t3-t0):7.2f} ms", flush=True)
# the drop-in path: mine() on a fresh host graph object (bench.py e2e)
from types import SimpleNamespace  # noqa: E402
plans = tmb.full_pattern_set(86400)
lab = np.full(g0.edge_count, -1, dtype=np.int8)
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    hg = SimpleNamespace(edge_src=hs, edge_dst=hd, edge_time=ht, node_count=g0.node_count, edge_label=lab)
    t0 = time.perf_counter()
    dg = tmb.as_device_graph(hg, 0)
    t1 = time.perf_counter()
    fm = tmb.mine(hg, plans)
    t2 = time.perf_counter()
    fm.device_graph.free()
    del fm, hg
    t3 = time.perf_counter()
    from paper_2604_12241_b200 import hostmem
    print(f"pool {hostmem.stats} ", end="")
    print(f"mine() rep {rep}: as_device_graph {1e3*(t1-t0):7.2f} ms  mine {1e3*(t2-t1):7.2f} ms  "
          f"free+del {1e3*(t3-t2):6.2f} ms  total {1e3*(t3-t0):7.2f} ms", flush=True)
