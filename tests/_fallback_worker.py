"""Runs in a subprocess with TM_LIB pointing at the tiny-caps test variant
(paper_2604_12241_b200/build.py TINY_DEFINES): mines graphs whose hub
windows overflow the tiny task queue, split-slot scratch, backward sets and
Bloom member lists, compares every column with the oracle, and prints the
work counters as JSON.  Test infrastructure (tests/test_gpu_fallbacks.py)."""

from __future__ import annotations

import ctypes
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2604_12241_b200 as tmb  # noqa: E402
from paper_2604_12241_b200 import _lib, synth  # noqa: E402
from oracle.oracle import OracleGraph, column  # noqa: E402


def counters(lib, reset=False):
    lib.tm_debug_counters.restype = ctypes.c_int
    lib.tm_debug_counters.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    buf = np.zeros(64, dtype=np.int64)
    n = lib.tm_debug_counters(1 if reset else 0, buf.ctypes.data, 64)
    return dict(zip(_lib.COUNTER_NAMES, buf[:n].tolist()))


def main():
    lib = _lib.load()
    counters(lib, reset=True)
    names = ["fan_in", "fan_out", "deg_in_src", "deg_out_dst", "cycle_2", "cycle_3", "cycle_4", "cycle_5",
             "cycle_6", "sg_count", "gs_count", "stack_count"]
    cases = [
        # long windows over alpha = 1 hubs: domain tasks, pull tasks, Bloom builds
        (synth.SynthConfig(2500, 50000, 8 * 86400, seed=23, powerlaw_exponent=1.0,
                           plants=(synth.PlantSpec("cycle_4", 20),)), 3 * 86400),
        # alpha = 2.1: one giant hub, many split rows
        (synth.SynthConfig(3000, 60000, 8 * 86400, seed=11, powerlaw_exponent=2.1,
                           plants=(synth.PlantSpec("sg_count", 40),)), 86400),
        # short windows (mean windowed degree < 2): the trigger kernel defers
        # chain descents and the tiny chain queue overflows into the rescue
        (synth.SynthConfig(4000, 80000, 30 * 86400, seed=5, powerlaw_exponent=1.0,
                           plants=(synth.PlantSpec("cycle_4", 40),)), 2 * 86400),
    ]
    bad = []
    for cfg, delta in cases:
        g0 = synth.generate(cfg)
        g = tmb.DeviceGraph(g0.src, g0.dst, g0.time)
        descs = [tmb.lower_plan(tmb.builtin_plan(n, delta)) for n in names]
        got = tmb.mine_rows(g, descs, 0, g.edge_count)  # host output: overflow -> whole call again
        want = OracleGraph(g0.src, g0.dst, g0.time).mine([column(n, delta) for n in names])
        bad += [f"{n}@{delta}" for j, n in enumerate(names) if not np.array_equal(got[:, j], want[:, j])]
        # device output: overflow -> gated inline rescue pass on the device
        import torch
        dev = torch.empty((g.edge_count, len(descs)), dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        tmb.mine_rows_device(g, descs, 0, g.edge_count, dev.data_ptr())
        torch.cuda.synchronize()
        got_d = dev.cpu().numpy()
        bad += [f"{n}@{delta}/device" for j, n in enumerate(names) if not np.array_equal(got_d[:, j], want[:, j])]
        g.free()
    print(json.dumps({"bad": bad, "counters": counters(lib)}))


if __name__ == "__main__":
    main()
