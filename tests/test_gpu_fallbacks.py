"""The exactness-preserving fallbacks of the mining kernels, driven on
purpose: a test build with tiny caps (build.py TINY_DEFINES: task queue 64,
split-row scratch 8, backward sets 3 nodes, Bloom member lists 8) mines
power-law graphs with long windows, and every column must still equal the
oracle while the work counters prove each fallback ran:

  queue_full   emit() / emit_whole() found the task queue full -> the warp
               walks the slice itself (tm_mine.cu emit)
  slot_full    no split-row scratch slot -> the warp walks the trigger's
               slices itself (k_mine_warp, slot = -2)
  useful_over  a backward set overflowed -> no pull candidates, the chain
               node is walked or split instead (useful_nodes)
  bloom_over   a Bloom layer's member list overflowed -> deeper layers are
               not built (treated as "all"), the walk stays exact
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("split", ["0", "1"])
def test_tiny_caps_variant_is_exact_and_hits_every_fallback(split):
    """split=1: item tasks defer their chain descents too (the big-call
    path, TM_SPLIT_TASKS) — their records overflow the tiny chain queue."""
    from paper_2604_12241_b200 import build
    lib = build.TINY_LIB
    assert lib.exists(), "build() makes the tiny-caps test variant"
    env = dict(os.environ, TM_LIB=str(lib), TM_SPLIT_TASKS=split)
    res = subprocess.run([sys.executable, str(ROOT / "tests" / "_fallback_worker.py")], env=env,
                         capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-4000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    assert out["bad"] == [], out
    c = out["counters"]
    for k in ("queue_full", "slot_full", "useful_over", "bloom_over", "chain_over"):
        assert c[k] > 0, (k, c)
