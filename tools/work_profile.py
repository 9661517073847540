"""Work profile of the mining kernels (GPU box): counts of items, windows,
bisection steps, membership probes and chain nodes per trigger.

    python tools/work_profile.py LIB.so [hi-small] [col ...]

LIB must be built with -DTM_COUNTERS=1 (build.build(defines=["TM_COUNTERS=1"])).
"""
import ctypes
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["TM_LIB"] = os.path.abspath(sys.argv[1])
import paper_2604_12241_b200 as tmb  # noqa: E402
from paper_2604_12241_b200 import _lib, synth  # noqa: E402

NAMES = _lib.COUNTER_NAMES

name = sys.argv[2] if len(sys.argv) > 2 else "hi-small"
cols = sys.argv[3:] or ["ALL14"]
lib = _lib.load()
fn = lib.tm_debug_counters
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_int]
buf = (ctypes.c_int64 * 64)()
g0 = synth.time_ordered(synth.generate(synth.CONFIGS[name]))
g = tmb.DeviceGraph(g0.src, g0.dst, g0.time, node_count=g0.node_count)
E = g.edge_count
for col in cols:
    descs = ([tmb.lower_plan(p) for p in tmb.full_pattern_set(86400)] if col == "ALL14"
             else [tmb.lower_plan(tmb.builtin_plan(col, 86400))])
    fn(1, buf, 64)
    tmb.mine_rows(g, descs, 0, E)
    n = fn(1, buf, 64)
    if n == 0:
        sys.exit("library built without TM_COUNTERS")
    print(f"== {name} {col}: E = {E}")
    for i in range(min(n, len(NAMES))):
        print(f"  {NAMES[i]:11s} {buf[i]:14d}  {buf[i] / E:9.3f} /trigger")
