"""The reference's own Python mining path, timed on sampled trigger blocks —
TEST INFRASTRUCTURE ONLY (bench.py's reference arm / cpu_baseline leg).

`oracle/stage_ref.sh` copies the reference package (`/root/reference/pkg/src
/tempmine`, pure Python + numpy) to `oracle/_ref/tempmine` (git-ignored, NOT
gpurun-ignored, so it travels to the GPU box; never imported by the product).
This module imports THAT copy, builds its `TemporalGraph` (txgraph.py:113-170)
from the same edge arrays the GPU gets, compiles the full pattern set with the
reference's own `compile_pattern` (plan.py:134: hinted builtins, GENERIC plans
for cycle_5/6 and gs_count from SURVEY Appendix B DSL), and times
`engine._mine_range(graph, plans, lo, hi, False)` (engine.py:607-646) — the
per-worker seam of `engine.mine` — over random contiguous 1000-trigger blocks
with a fork pool of os.cpu_count() workers, like `mine(workers=P)`
(engine.py:677-690).  The full HI-* runs do not finish in minutes (SURVEY
§8d), so the edges/s figure is EXTRAPOLATED from the blocks.  The rows it
returns are the reference's own counts: bench.py also compares the GPU
output with them (parity against the reference itself, not the port).
"""

from __future__ import annotations

import multiprocessing
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"


def available() -> bool:
    return (REF_DIR / "tempmine" / "engine.py").exists()


def _import():
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import tempmine.dsl as dsl  # noqa: F401
    import tempmine.engine as engine
    import tempmine.plan as plan
    import tempmine.txgraph as txgraph
    return dsl, engine, plan, txgraph


# SURVEY Appendix B DSL (the same texts tests/golden/make_golden.py uses)
def _cycle_k_text(k: int, delta: int) -> str:
    chain = k - 3
    lines = [f"pattern: cycle_{k}", f"delta: {delta}", ""]
    for i in range(1, chain + 1):
        lines += ["stage:", "  op: for_all", f"  src: {'N1' if i == 1 else f'A{i-1}'}.out_neigh", f"  dst_var: A{i}"]
        if i == 1:
            lines.append("  skip_if: N0 == N1")
        lines.append(f"  skip_if: A{i} == N0")
        if i >= 2:
            lines.append(f"  skip_if: A{i} == N1")
        lines += [f"  skip_if: A{i} == A{j}" for j in range(1, i - 1)]
        lines.append("")
    lines += ["stage:", "  op: intersect", f"  src: A{chain}.out_neigh, N0.in_neigh", "  dst_var: C",
              "  skip_if: C == N1"]
    lines += [f"  skip_if: C == A{j}" for j in range(1, chain)]
    lines += ["", "emit:", "  mode: set_cardinality", "  target: C"]
    return "\n".join(lines) + "\n"


def _gs_text(delta: int) -> str:
    return (f"pattern: gs_count\ndelta: {delta}\n\n"
            "stage:\n  op: for_all\n  src: N1.out_neigh\n  dst_var: D\n  skip_if: D == N0\n\n"
            "stage:\n  op: intersect\n  src: D.in_neigh, N0.out_neigh\n  dst_var: M\n\n"
            "emit:\n  mode: source_count\n  min_size: 2\n  target: M\n")


def reference_plans(names, delta: int, stats=None):
    """The reference's compiled ExecutionPlans for column `names`, in that order."""
    import dataclasses
    dsl, _, plan, _ = _import()
    out = []
    for n in names:
        if n in plan.BUILTIN_COLUMNS:
            vp = plan.load_builtin(n)
            vp = dsl.must_validate(dataclasses.replace(vp.spec, delta=delta))
        elif n == "gs_count":
            vp = dsl.must_validate(dsl.parse_pattern(_gs_text(delta)))
        elif n.startswith("cycle_") and int(n.split("_")[1]) >= 5:
            vp = dsl.must_validate(dsl.parse_pattern(_cycle_k_text(int(n.split("_")[1]), delta)))
        else:
            raise ValueError(f"no reference pattern for column {n!r}")
        out.append(plan.compile_pattern(vp, stats))
    return out


_CTX: dict = {}


def _block(b):
    lo, hi = b
    t = time.perf_counter()
    block, _, _ = _CTX["engine"]._mine_range(_CTX["graph"], _CTX["plans"], lo, hi, False)
    return block, time.perf_counter() - t


class RefPython:
    """The reference's TemporalGraph + plans; mine(blocks) with a fork pool."""

    def __init__(self, src, dst, t, node_count: int, names, delta: int):
        _, engine, _, txgraph = _import()
        E = len(src)
        t0 = time.perf_counter()
        self.graph = txgraph.TemporalGraph(
            node_count=int(node_count), edge_src=np.asarray(src, dtype=np.int64),
            edge_dst=np.asarray(dst, dtype=np.int64), edge_time=np.asarray(t, dtype=np.int64),
            edge_amount=np.zeros(E, dtype=np.float64), edge_currency=np.zeros(E, dtype=np.int32),
            edge_label=np.full(E, -1, dtype=np.int8), currency_vocab=("USD",))
        self.build_s = time.perf_counter() - t0
        self.engine = engine
        self.plans = reference_plans(names, delta, self.graph.stats)
        self.names = list(names)

    def mine(self, blocks, workers: int | None = None):
        """(rows per block, summed per-block seconds, wall seconds) over a
        fork pool of `workers` (default os.cpu_count())."""
        workers = workers or os.cpu_count() or 1
        _CTX.update(engine=self.engine, graph=self.graph, plans=self.plans)
        t = time.perf_counter()
        try:
            if workers == 1:
                res = [_block(b) for b in blocks]
            else:
                with multiprocessing.get_context("fork").Pool(workers) as pool:
                    res = pool.map(_block, blocks, chunksize=1)
        finally:
            _CTX.clear()
        wall = time.perf_counter() - t
        return [r[0] for r in res], float(sum(r[1] for r in res)), wall
