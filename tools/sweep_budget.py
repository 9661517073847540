"""Light-tier budget sweep (GPU box): python tools/sweep_budget.py [hi-small]
Each budget runs in a fresh process (TM_LIGHT_BUDGET is read once)."""
import os
import subprocess
import sys

name = sys.argv[1] if len(sys.argv) > 1 else "hi-small"
code = r'''
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2604_12241_b200 as tmb
from paper_2604_12241_b200 import _lib, synth
g0 = synth.time_ordered(synth.generate(synth.CONFIGS[sys.argv[1]]))
g = tmb.DeviceGraph(g0.src, g0.dst, g0.time, node_count=g0.node_count)
_lib.check(_lib.load().tm_set_profiling(g.handle, 1), "prof")
descs = [tmb.lower_plan(p) for p in tmb.full_pattern_set(86400)]
best = None
for rep in range(4):
    out = tmb.mine_rows(g, descs, 0, g.edge_count)
    st = tmb.last_stats(g)
    t = st.total_ms
    if best is None or t < best[0]:
        best = (t, st.light_ms, st.heavy_ms, st.heavy_triggers)
import os
print(f"budget {sys.argv[2]:>5s} chunks {os.environ.get('TM_CHUNKS', 'auto'):>4s}: wall {best[0]:7.3f} ms  light-sum {best[1]:7.3f}  heavy-sum {best[2]:7.3f}  heavy_n {best[3]}  sum {int(out.sum())}", flush=True)
'''
for spec in sys.argv[2:] or ["64", "96", "160"]:
    b, _, ch = spec.partition(":")
    env = dict(os.environ, TM_LIGHT_BUDGET=b)
    if ch:
        env["TM_CHUNKS"] = ch
    subprocess.run([sys.executable, "-c", code, name, b], env=env, check=False)
