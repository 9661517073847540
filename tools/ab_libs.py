"""A/B timing of library variants on the GPU box.

    python tools/ab_libs.py hi-small lib_a.so lib_b.so ...

The workload is generated once (/tmp cache); each library runs in a fresh
process (TM_LIB=path): full 14-column set at
delta 86400, device-resident output, best of 5 device-timed calls, plus a
checksum so variants are compared on identical results.
"""
import os
import subprocess
import sys

CODE = r'''
import sys, json
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2604_12241_b200 as tmb
from paper_2604_12241_b200 import _lib, synth
z = np.load(sys.argv[3])
g = tmb.DeviceGraph(z["src"], z["dst"], z["time"], node_count=int(z["n"]))
_lib.check(_lib.load().tm_set_profiling(g.handle, 1), "prof")
descs = [tmb.lower_plan(p) for p in tmb.full_pattern_set(86400)]
E = g.edge_count
out = torch.empty((E, len(descs)), dtype=torch.int64, device="cuda")
st_ = torch.cuda.Stream()
best = None
for rep in range(6):
    tmb.mine_rows_device(g, descs, 0, E, out.data_ptr(), st_.cuda_stream)
    s = tmb.last_stats(g)
    if rep and (best is None or s.total_ms < best[0]):
        best = (s.total_ms, s.light_ms, s.heavy_ms)
torch.cuda.synchronize()
cs = [int(x) for x in out.sum(dim=0).tolist()]
print(json.dumps({"lib": sys.argv[2], "config": sys.argv[1], "ms": round(best[0], 3),
                  "warp_ms": round(best[1], 3), "task_ms": round(best[2], 3),
                  "edges_per_s": E / best[0] * 1e3, "colsums": cs}), flush=True)
'''

cfg = sys.argv[1]
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
from paper_2604_12241_b200 import synth  # noqa: E402
cache = f"/tmp/ab_{cfg}.npz"
if not os.path.exists(cache):  # generate once for every variant
    g0 = synth.time_ordered(synth.generate(synth.CONFIGS[cfg]))
    np.savez(cache, src=g0.src, dst=g0.dst, time=g0.time, n=g0.node_count)
for lib in sys.argv[2:]:
    env = dict(os.environ, TM_LIB=os.path.abspath(lib))
    subprocess.run([sys.executable, "-c", CODE, cfg, os.path.basename(lib), cache], env=env, check=False)
