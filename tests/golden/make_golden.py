"""Generate the golden parity fixtures by running the REFERENCE itself.

Run in the build container only (the reference is mounted read-only at
/root/reference; it does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every expected value in tests/golden/*.npz / *.json comes from
`tempmine.engine.mine` (engine.py:658) — hinted batch kernels for the 11
builtins (kernels.py:290-402) and the generic interpreter
(engine.py:516-562) for the extended families (cycle_5..8, gs_count), whose
DSL is SURVEY.md Appendix B. Nothing here is produced by this repo's code.

Fixtures:
  hand_cases.json  the reference unit tests' known-answer graphs
                   (test_kernels.py, test_oracle.py, test_engine.py) mined
                   with every column
  corpus.npz       acceptance corpus C1 (test_acceptance.py:44-61,
                   CORPUS_SEED=20260808), all 200 graphs x 3 deltas
  ties.npz         random graphs with self-loops and heavy timestamp ties
  cfg1.npz         SURVEY §8d cfg1: synth.generate(10K nodes, 100K bg txns,
                   16 d horizon, seed 7, planted) at delta=86400 — arrays
                   pinned by sha256 so paper_2604_12241_b200.synth can be
                   checked bit-for-bit against synth.generate
"""

from __future__ import annotations

import dataclasses
import hashlib
import json
import multiprocessing
import os
import random
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, "/root/reference/pkg")

from tempmine import dsl, plan, synth  # noqa: E402
from tempmine.engine import mine  # noqa: E402
from tempmine.plan import BUILTIN_COLUMNS, compile_pattern  # noqa: E402
from tempmine.txgraph import TemporalGraph, TransactionRecord, build_graph  # noqa: E402

OUT = Path(__file__).resolve().parent


# ---------------------------------------------------------------------------
# Extended-family DSL — written here from the grammar


def cycle_k_text(k: int, delta: int, min_size: int = 1, name: str | None = None) -> str:
    assert 5 <= k <= 8
    chain = k - 3
    lines = [f"pattern: {name or f'cycle_{k}'}", f"delta: {delta}", ""]
    for i in range(1, chain + 1):
        lines.append("stage:")
        lines.append("  op: for_all")
        lines.append(f"  src: {'N1' if i == 1 else f'A{i-1}'}.out_neigh")
        lines.append(f"  dst_var: A{i}")
        if i == 1:
            lines.append("  skip_if: N0 == N1")
        lines.append(f"  skip_if: A{i} == N0")
        if i >= 2:
            lines.append(f"  skip_if: A{i} == N1")
        for j in range(1, i - 1):
            lines.append(f"  skip_if: A{i} == A{j}")
        lines.append("")
    lines.append("stage:")
    lines.append("  op: intersect")
    lines.append(f"  src: A{chain}.out_neigh, N0.in_neigh")
    lines.append("  dst_var: C")
    lines.append("  skip_if: C == N1")
    for j in range(1, chain):
        lines.append(f"  skip_if: C == A{j}")
    lines.append("")
    lines.append("emit:")
    lines.append("  mode: set_cardinality")
    if min_size != 1:
        lines.append(f"  min_size: {min_size}")
    lines.append("  target: C")
    return "\n".join(lines) + "\n"


def gs_text(delta: int, min_size: int = 2, name: str = "gs_count") -> str:
    return (f"pattern: {name}\ndelta: {delta}\n\n"
            "stage:\n  op: for_all\n  src: N1.out_neigh\n  dst_var: D\n  skip_if: D == N0\n\n"
            "stage:\n  op: intersect\n  src: D.in_neigh, N0.out_neigh\n  dst_var: M\n\n"
            f"emit:\n  mode: source_count\n  min_size: {min_size}\n  target: M\n")


def builtin_with(name: str, delta: int, min_size: int | None = None,
                 new_name: str | None = None, attribution: str = "trigger") -> dsl.ValidatedPattern:
    vp = plan.load_builtin(name)
    spec = dataclasses.replace(vp.spec, delta=delta, attribution=attribution)
    if min_size is not None:
        spec = dataclasses.replace(spec, emit=dataclasses.replace(spec.emit, min_size=min_size))
    if new_name is not None:
        spec = dataclasses.replace(spec, name=new_name)
    return dsl.must_validate(spec)


def ext_pattern(base: str, delta: int, min_size: int | None, name: str,
                attribution: str = "trigger") -> dsl.ValidatedPattern:
    if base == "gs_count":
        text = gs_text(delta, 2 if min_size is None else min_size, name)
    else:
        text = cycle_k_text(int(base.split("_")[1]), delta, 1 if min_size is None else min_size, name)
    if attribution != "trigger":
        text = text.replace("\n\nstage:", f"\nattribution: {attribution}\n\nstage:", 1)
    return dsl.must_validate(dsl.parse_pattern(text))


# column spec: (column name, family base name, min_size or None=default)
BUILTIN_SPECS = [(n, n, None) for n in BUILTIN_COLUMNS]
EXT_SPECS = [("cycle_5", "cycle_5", None), ("cycle_6", "cycle_6", None),
             ("cycle_7", "cycle_7", None), ("cycle_8", "cycle_8", None),
             ("gs_count", "gs_count", None)]
VARIANT_SPECS = [("sg_k1", "sg_count", 1), ("sg_k3", "sg_count", 3),
                 ("gs_k1", "gs_count", 1), ("fan_in_k2", "fan_in", 2),
                 ("deg_out_src_k3", "deg_out_src", 3), ("cycle_2_k2", "cycle_2", 2),
                 ("cycle_3_k2", "cycle_3", 2), ("cycle_4_k2", "cycle_4", 2),
                 ("cycle_5_k2", "cycle_5", 2), ("stack_k2", "stack_count", 2)]
ALL_SPECS = BUILTIN_SPECS + EXT_SPECS + VARIANT_SPECS


def patterns_for(specs, delta: int, attribution: str = "trigger"):
    out = []
    for col, base, k in specs:
        if base in BUILTIN_COLUMNS:
            out.append(builtin_with(base, delta, k, None if col == base else col, attribution))
        else:
            out.append(ext_pattern(base, delta, k, col, attribution))
    return out


def mine_columns(g: TemporalGraph, specs, delta: int, workers: int = 1,
                 attribution: str = "trigger") -> np.ndarray:
    pats = patterns_for(specs, delta, attribution)
    plans = [compile_pattern(p, g.stats) for p in pats]
    fm = mine(g, plans, workers=workers)
    return np.stack([fm.column(col) for col, _, _ in specs], axis=1).astype(np.int64)


def graph_from_edges(edges) -> TemporalGraph:
    recs = [TransactionRecord(i, e[0], e[1], e[2], 100.0, "SYN") for i, e in enumerate(edges)]
    return build_graph(recs)


def graph_from_arrays(src, dst, t) -> TemporalGraph:
    n = int(max(src.max(), dst.max())) + 1
    e = len(src)
    return TemporalGraph(n, src.astype(np.int64), dst.astype(np.int64), t.astype(np.int64),
                         np.full(e, 100.0), np.zeros(e, dtype=np.int32),
                         np.full(e, -1, dtype=np.int8), ("SYN",))


def spec_json(specs):
    return [{"column": c, "base": b, "min_size": k} for c, b, k in specs]


# ---------------------------------------------------------------------------
# hand cases: the reference's known-answer graphs


HAND_GRAPHS = {
    # test_kernels.py
    "fan_star": ([(i, 5, i + 1) for i in range(5)], [10, 0, 2]),
    "isolated": ([(0, 1, 5)], [10, 0]),
    "parallel_fan": ([(0, 1, 5), (0, 1, 5), (2, 1, 4)], [10, 0]),
    "fan_selfloop": ([(1, 1, 4), (0, 1, 5)], [10, 0, 1]),
    "deg_single": ([(0, 1, 7)], [5]),
    "deg_reverse": ([(1, 0, 3), (0, 1, 5)], [5, 1]),
    "cycle4": ([(0, 1, 1), (1, 2, 2), (2, 3, 3), (3, 0, 4)], [10, 2, 0]),
    "cycle2": ([(0, 1, 1), (1, 0, 2)], [5, 0]),
    "triangle": ([(0, 1, 1), (1, 2, 2), (2, 0, 3)], [10]),
    "node_tuples": ([(0, 1, 5), (1, 0, 3), (1, 0, 4)], [10]),
    "cycle4_scrambled": ([(0, 1, 1), (1, 2, 3), (2, 3, 2), (3, 0, 4)], [10]),
    "selfloop_trigger_cycles": ([(0, 0, 5), (0, 1, 3), (1, 0, 4)], [10]),
    "sg_planted": ([(0, 2, 1), (0, 3, 2), (0, 4, 3), (2, 1, 4), (3, 1, 5), (4, 1, 6)], [10, 3]),
    "sg_ordered": ([(0, 1, 4), (1, 2, 5), (0, 3, 4), (3, 2, 2)], [10]),
    "stack_one_each": ([(2, 0, 1), (0, 1, 2), (1, 3, 1)], [5]),
    "stack_no_upstream": ([(0, 1, 2), (1, 3, 1)], [5]),
    "stack_forward": ([(2, 0, 1), (0, 1, 2), (1, 3, 1), (1, 4, 3)], [5]),
    "windowed_nodes_loops": ([(0, 0, 5), (0, 1, 5), (0, 2, 9)], [10, 4]),
    # SURVEY Appendix A exactness traps
    "same_tick_larger_eid": ([(0, 1, 5), (1, 0, 5), (2, 0, 5)], [0, 3]),
    "selfloop_trigger_stack": ([(0, 0, 5), (1, 0, 4), (0, 2, 4)], [10]),
    "parallel_cycle3": ([(1, 2, 1), (1, 2, 2), (2, 0, 3), (2, 0, 3), (0, 1, 4)], [10]),
    # test_engine.py zero-delta on strictly increasing times
    "zero_delta_increasing": ([(i % 5, (i * 3 + 1) % 5, i) for i in range(20)
                               if i % 5 != (i * 3 + 1) % 5], [0]),
    # 5..8-cycles through the trigger, and a gather-scatter
    "cycle5": ([(0, 1, 1), (1, 2, 2), (2, 3, 3), (3, 4, 4), (4, 0, 5)], [10, 3]),
    "cycle6": ([(i, (i + 1) % 6, i + 1) for i in range(6)], [10]),
    "cycle7": ([(i, (i + 1) % 7, i + 1) for i in range(7)], [10]),
    "cycle8": ([(i, (i + 1) % 8, i + 1) for i in range(8)] + [(3, 6, 2), (6, 0, 3)], [10, 5]),
    "gs_planted": ([(5, 2, 1), (5, 3, 2), (7, 2, 3), (7, 3, 4), (0, 5, 5), (0, 7, 5),
                    (1, 7, 6), (0, 1, 7)], [10, 2]),
    "cycle5_selfloop_chain": ([(0, 1, 1), (1, 1, 2), (1, 2, 2), (2, 3, 3), (3, 4, 4),
                               (4, 0, 5), (4, 0, 5), (2, 2, 3)], [10]),
}


def make_hand():
    cases = []
    for name, (edges, deltas) in HAND_GRAPHS.items():
        g = graph_from_edges(edges)
        for delta in deltas:
            vals = mine_columns(g, ALL_SPECS, delta)
            cases.append({"name": name, "edges": [list(e) for e in edges], "delta": delta,
                          "values": vals.tolist()})
    doc = {"generator": "tests/golden/make_golden.py", "reference": "tempmine 0.1.0 (engine.mine)",
           "columns": spec_json(ALL_SPECS), "cases": cases}
    (OUT / "hand_cases.json").write_text(json.dumps(doc, separators=(",", ":")) + "\n")
    print(f"hand_cases.json: {len(cases)} cases")


# ---------------------------------------------------------------------------
# acceptance corpus (test_acceptance.py:44-61)

CORPUS_SEED = 20260808


def corpus_params():
    rng = random.Random(CORPUS_SEED)
    params = []
    for _ in range(200):
        n_nodes = rng.randint(6, 50)
        n_edges = rng.randint(15, 400)
        horizon = rng.randint(8, 2000)
        deltas = (rng.randint(0, max(horizon // 10, 1)), rng.randint(1, horizon),
                  rng.randint(horizon, 2 * horizon))
        params.append((rng.randrange(2 ** 31), n_nodes, n_edges, horizon, deltas))
    s0, *_, d0 = params[0]
    params[0] = (s0, 50, 400, 600, d0)
    s1, *_, _ = params[1]
    params[1] = (s1, 50, 400, 9, (0, 3, 11))
    return params


def corpus_records(seed, n_nodes, n_edges, horizon):
    # conftest.random_records (selfloops allowed)
    rng = random.Random(seed)
    out = []
    for _ in range(n_edges):
        u = rng.randrange(n_nodes)
        v = rng.randrange(n_nodes)
        out.append((u, v, rng.randrange(horizon)))
    return out


# cycle_6..8 are left out of the dense corpus: the reference's generic
# interpreter needs hours on 50-node / 400-edge whole-graph windows.  They are
# pinned on the sparse `ties` graphs, the hand cases and cfg1 instead.
CORPUS_SPECS = [s for s in ALL_SPECS if s[0] not in ("cycle_6", "cycle_7", "cycle_8")]


def _corpus_one(p):
    seed, n_nodes, n_edges, horizon, deltas = p
    edges = corpus_records(seed, n_nodes, n_edges, horizon)
    g = graph_from_edges(edges)
    vals = [mine_columns(g, CORPUS_SPECS, d) for d in deltas]
    return np.array(edges, dtype=np.int64), np.array(deltas, dtype=np.int64), np.stack(vals)


def make_corpus():
    params = corpus_params()
    with multiprocessing.get_context("fork").Pool(os.cpu_count()) as pool:
        res = pool.map(_corpus_one, params, chunksize=1)
    edges = np.concatenate([r[0] for r in res])
    offsets = np.cumsum([0] + [len(r[0]) for r in res]).astype(np.int64)
    deltas = np.stack([r[1] for r in res])
    vals = np.concatenate([r[2].transpose(1, 0, 2) for r in res])  # (sumE, 3, C)
    assert vals.max() < 2 ** 31
    np.savez_compressed(OUT / "corpus.npz", edges=edges.astype(np.int32), offsets=offsets,
                        deltas=deltas, values=vals.astype(np.int32),
                        columns=json.dumps(spec_json(CORPUS_SPECS)))
    print(f"corpus.npz: {len(params)} graphs, {len(edges)} edges")


# ---------------------------------------------------------------------------
# self-loops + timestamp ties at moderate size


TIES_CASES = [  # (seed, n_nodes, n_edges, horizon, deltas)
    (11, 400, 6000, 60, (0, 2, 9)),
    (12, 2000, 20000, 2000, (0, 30, 200)),
]


def make_ties():
    arrays = {}
    meta = []
    for idx, (seed, n, e, h, deltas) in enumerate(TIES_CASES):
        rng = np.random.Generator(np.random.PCG64(seed))
        # skewed sources (a few hubs) + uniform dst; self-loops allowed
        w = np.arange(1, n + 1, dtype=np.float64) ** -1.2
        w /= w.sum()
        src = rng.choice(n, size=e, p=w)
        dst = rng.integers(0, n, size=e)
        loops = rng.random(e) < 0.03
        dst[loops] = src[loops]
        t = rng.integers(0, h, size=e)
        g = graph_from_arrays(src, dst, t)
        vals = np.stack([mine_columns(g, ALL_SPECS, d, workers=os.cpu_count()) for d in deltas], axis=1)
        arrays[f"src{idx}"] = src.astype(np.int32)
        arrays[f"dst{idx}"] = dst.astype(np.int32)
        arrays[f"time{idx}"] = t.astype(np.int32)
        arrays[f"values{idx}"] = vals
        meta.append({"seed": seed, "n_nodes": n, "n_edges": e, "horizon": h, "deltas": list(deltas)})
        print(f"ties case {idx}: done")
    np.savez_compressed(OUT / "ties.npz", meta=json.dumps(meta),
                        columns=json.dumps(spec_json(ALL_SPECS)), **arrays)


# ---------------------------------------------------------------------------
# cfg1


CFG1 = dict(node_count=10_000, background_edge_count=100_000, time_horizon=16 * 86400, seed=7)
CFG1_PLANTS = (synth.PlantSpec("sg_count", 100), synth.PlantSpec("cycle_2", 50),
               synth.PlantSpec("cycle_3", 50), synth.PlantSpec("cycle_4", 50),
               synth.PlantSpec("stack_count", 50))
CFG1_SPECS = BUILTIN_SPECS + EXT_SPECS


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def make_cfg1():
    cfg = synth.SynthConfig(**CFG1, plants=CFG1_PLANTS)
    records, truth = synth.generate(cfg)
    g = build_graph(records)
    t0 = time.time()
    vals = mine_columns(g, CFG1_SPECS, 86400, workers=os.cpu_count())
    print(f"cfg1 mined in {time.time() - t0:.1f}s")
    # unplanted background only, as in the survey's per-builtin sums
    cfg0 = synth.SynthConfig(**CFG1)
    rec0, _ = synth.generate(cfg0)
    g0 = build_graph(rec0)
    sums0 = mine_columns(g0, BUILTIN_SPECS, 86400, workers=os.cpu_count()).sum(axis=0)
    np.savez_compressed(
        OUT / "cfg1.npz", values=vals, columns=json.dumps(spec_json(CFG1_SPECS)),
        sha_src=sha(g.edge_src), sha_dst=sha(g.edge_dst), sha_time=sha(g.edge_time),
        node_count=g.node_count, edge_count=g.edge_count,
        head=np.stack([g.edge_src[:64], g.edge_dst[:64], g.edge_time[:64]]),
        tail=np.stack([g.edge_src[-64:], g.edge_dst[-64:], g.edge_time[-64:]]),
        truth_triggers=np.array([r.trigger_edge for r in truth], dtype=np.int64),
        unplanted_sums=sums0, unplanted_sha_src=sha(g0.edge_src),
        unplanted_sha_dst=sha(g0.edge_dst), unplanted_sha_time=sha(g0.edge_time))
    print("cfg1.npz written; unplanted sums:", dict(zip(BUILTIN_COLUMNS, sums0.tolist())))


# ---------------------------------------------------------------------------
# compiled reference plans (plan.py:134-187), for the drop-in lowering tests


CUSTOM_DIR = Path("/root/reference/pkg/tests/data/custom")
CUSTOM_NAMES = ("spray_union", "filtered_senders", "sg_ordered", "stack_forward", "chain_5cycle")


# ---------------------------------------------------------------------------
# members attribution (engine.py:629-640, pattern_grammar.md:116-122): an
# instance is anchored at its temporally last member edge and adds 1 to the
# row of every member edge


def _corpus_one_members(p):
    seed, n_nodes, n_edges, horizon, deltas = p
    edges = corpus_records(seed, n_nodes, n_edges, horizon)
    g = graph_from_edges(edges)
    vals = [mine_columns(g, CORPUS_SPECS, d, attribution="members") for d in deltas]
    return np.stack(vals)


def make_members():
    cases = []
    for name, (edges, deltas) in HAND_GRAPHS.items():
        g = graph_from_edges(edges)
        for delta in deltas:
            vals = mine_columns(g, ALL_SPECS, delta, attribution="members")
            cases.append({"name": name, "edges": [list(e) for e in edges], "delta": delta,
                          "values": vals.tolist()})
    doc = {"generator": "tests/golden/make_golden.py", "reference": "tempmine 0.1.0 (engine.mine)",
           "attribution": "members", "columns": spec_json(ALL_SPECS), "cases": cases}
    (OUT / "hand_members.json").write_text(json.dumps(doc, separators=(",", ":")) + "\n")
    print(f"hand_members.json: {len(cases)} cases")
    params = corpus_params()
    with multiprocessing.get_context("fork").Pool(os.cpu_count()) as pool:
        res = pool.map(_corpus_one_members, params, chunksize=1)
    vals = np.concatenate([r.transpose(1, 0, 2) for r in res])
    assert vals.max() < 2 ** 31
    np.savez_compressed(OUT / "corpus_members.npz", values=vals.astype(np.int32),
                        columns=json.dumps(spec_json(CORPUS_SPECS)))
    print("corpus_members.npz written (edges/deltas: corpus.npz)")
    seed, n, e, h, deltas = TIES_CASES[0]
    z = np.load(OUT / "ties.npz")
    g = graph_from_arrays(z["src0"].astype(np.int64), z["dst0"].astype(np.int64), z["time0"].astype(np.int64))
    tv = np.stack([mine_columns(g, ALL_SPECS, d, workers=os.cpu_count(), attribution="members")
                   for d in deltas], axis=1)
    np.savez_compressed(OUT / "ties_members.npz", values0=tv, columns=json.dumps(spec_json(ALL_SPECS)))
    print("ties_members.npz written (case 0)")


def make_cfg1_members():
    cfg = synth.SynthConfig(**CFG1, plants=CFG1_PLANTS)
    records, _ = synth.generate(cfg)
    g = build_graph(records)
    specs = BUILTIN_SPECS + [("cycle_5", "cycle_5", None), ("gs_count", "gs_count", None)]
    t0 = time.time()
    vals = mine_columns(g, specs, 86400, workers=os.cpu_count(), attribution="members")
    print(f"cfg1 members mined in {time.time() - t0:.1f}s")
    np.savez_compressed(OUT / "cfg1_members.npz", values=vals, columns=json.dumps(spec_json(specs)))


def make_plans():
    entries = []
    for col, base, k in ALL_SPECS:
        vp = patterns_for([(col, base, k)], 3600)[0]
        for forced in (False, True):
            p = compile_pattern(vp, None, force_generic=forced)
            entries.append({"column": col, "base": base, "min_size": k, "force_generic": forced,
                            "plan": dataclasses.asdict(p)})
    for name in CUSTOM_NAMES:
        vp = dsl.must_validate(dsl.parse_pattern((CUSTOM_DIR / f"{name}.pat").read_text()))
        p = compile_pattern(vp, None)
        entries.append({"column": name, "base": None, "min_size": None, "force_generic": False,
                        "plan": dataclasses.asdict(p)})
    (OUT / "plans.json").write_text(json.dumps({"generator": "tests/golden/make_golden.py",
                                                "plans": entries}, indent=0) + "\n")
    print(f"plans.json: {len(entries)} plans")


# ---------------------------------------------------------------------------
# instance lists (mine(..., collect_instances=True), engine.py:629-645,
# 658-720): every instance _EmissionState records (engine.py:455-513) as
# InstanceRecord(pattern, trigger_edge, sorted member_edges, sorted
# member_nodes), sorted by (pattern, trigger_edge, member_edges).  Stored as
# one int32 stream per case: [pattern index, trigger, n_edges, n_nodes,
# edges..., nodes...] per record, in the reference's order.

INSTANCE_CORPUS = 24      # first graphs of the acceptance corpus, smallest delta


def collect_records(g: TemporalGraph, specs, delta: int, workers: int = 1) -> np.ndarray:
    pats = patterns_for(specs, delta)
    plans = [compile_pattern(p, g.stats) for p in pats]
    _, inst = mine(g, plans, workers=workers, collect_instances=True)
    col = {c: i for i, (c, _, _) in enumerate(specs)}
    out = []
    for r in inst:
        out += [col[r.pattern], r.trigger_edge, len(r.member_edges), len(r.member_nodes)]
        out += list(r.member_edges) + list(r.member_nodes)
    return np.array(out, dtype=np.int32)


def _corpus_one_instances(p):
    seed, n_nodes, n_edges, horizon, deltas = p
    edges = corpus_records(seed, n_nodes, n_edges, horizon)
    g = graph_from_edges(edges)
    return collect_records(g, CORPUS_SPECS, int(deltas[0]))


def make_instances():
    arrays, meta = {}, []
    for name, (edges, deltas) in HAND_GRAPHS.items():
        g = graph_from_edges(edges)
        for delta in deltas:
            arrays[f"rec{len(meta)}"] = collect_records(g, ALL_SPECS, delta)
            arrays[f"edges{len(meta)}"] = np.array(edges, dtype=np.int64).reshape(-1, 3)
            meta.append({"name": name, "delta": delta, "specs": "all"})
    params = corpus_params()[:INSTANCE_CORPUS]
    with multiprocessing.get_context("fork").Pool(os.cpu_count()) as pool:
        res = pool.map(_corpus_one_instances, params, chunksize=1)
    for i, (p, rec) in enumerate(zip(params, res)):
        seed, n_nodes, n_edges, horizon, deltas = p
        arrays[f"rec{len(meta)}"] = rec
        arrays[f"edges{len(meta)}"] = np.array(corpus_records(seed, n_nodes, n_edges, horizon),
                                               dtype=np.int64)
        meta.append({"name": f"corpus{i}", "delta": int(deltas[0]), "specs": "corpus"})
    z = np.load(OUT / "ties.npz")  # self-loops + same-tick ties, delta 0
    src, dst, t = (z[f"{k}0"].astype(np.int64) for k in ("src", "dst", "time"))
    arrays[f"rec{len(meta)}"] = collect_records(graph_from_arrays(src, dst, t), ALL_SPECS, 0,
                                                workers=os.cpu_count())
    arrays[f"edges{len(meta)}"] = np.stack([src, dst, t], axis=1)
    meta.append({"name": "ties0", "delta": 0, "specs": "all"})
    n = sum(len(a) for k, a in arrays.items() if k.startswith("rec"))
    np.savez_compressed(OUT / "instances.npz", meta=json.dumps(meta),
                        all_columns=json.dumps(spec_json(ALL_SPECS)),
                        corpus_columns=json.dumps(spec_json(CORPUS_SPECS)), **arrays)
    print(f"instances.npz: {len(meta)} cases, {n} record words")


# ---------------------------------------------------------------------------
# GENERIC stage programs: the reference's shipped custom
# patterns (tests/data/custom/*.pat) plus programs written here from the
# grammar (pattern_grammar.md) to reach every interpreter feature: union /
# differentiate, set references (bound X.self, siblings), 3-deep nests,
# forward windows, order constraints (with t), edge-identity, amount and
# currency predicates, gates on e0 and on an enclosing symbol, every
# emission mode, min_size > 1.  Expected values: tempmine.engine.mine on
# compile_pattern(force_generic=True) plans.

VM_PATTERNS = {
    "union3": """pattern: union3
delta: {delta}
stage:
  op: union
  src: N0.out_neigh, N1.out_neigh, N1.in_neigh
  dst_var: U
  skip_if: U == N0
emit:
  mode: set_cardinality
  target: U
""",
    "fwd_fan": """pattern: fwd_fan
delta: {delta}
stage:
  op: for_all
  src: N1.out_neigh
  dst_var: F
  window: forward
  skip_if: e1 == e0
  break_if: e1.t > t + delta
emit:
  mode: edge_count
  min_size: 2
  target: F
""",
    "ord_cycle3": """pattern: ord_cycle3
delta: {delta}
stage:
  op: for_all
  src: N1.out_neigh
  dst_var: A
  skip_if: A == N0
stage:
  op: intersect
  src: A.out_neigh, N0.in_neigh
  dst_var: C
  skip_if: C == N1
  order: e1.t <= e2.t
  order: e2.t <= e3.t
  order: e3.t <= t
emit:
  mode: set_cardinality
  target: C
""",
    "big_out": """pattern: big_out
delta: {delta}
stage:
  op: for_all
  src: N0.out_neigh
  dst_var: X
  skip_if: e1.amount < 500
  skip_if: e1 == e0
emit:
  mode: instance_list
  target: X
""",
    "gate_cur": """pattern: gate_cur
delta: {delta}
stage:
  op: for_all
  src: N1.in_neigh
  dst_var: S
  skip_if: e0.amount > 700
  skip_if: e1.currency != "USD"
emit:
  mode: set_cardinality
  target: S
""",
    "same_cur_stack": """pattern: same_cur_stack
delta: {delta}
stage:
  op: for_all
  src: N0.in_neigh
  dst_var: A
  skip_if: e1.currency != e0.currency
  skip_if: A == N1
stage:
  op: for_all
  src: N1.out_neigh
  dst_var: C
  window: forward
  skip_if: e2.currency > e0.currency
  skip_if: C == N0
emit:
  mode: pair_product
  target: A, C
""",
    "nest_self": """pattern: nest_self
delta: {delta}
stage:
  op: for_all
  src: N1.out_neigh
  dst_var: A
  skip_if: A == N0
stage:
  op: for_all
  src: A.out_neigh
  dst_var: B
  skip_if: B == N1
  skip_if: B == N0
stage:
  op: intersect
  src: B.out_neigh, A.self
  dst_var: C
stage:
  op: differentiate
  src: C.self
  dst_var: D
  skip_if: D == N1
emit:
  mode: source_count
  target: D
""",
    "gate_anc": """pattern: gate_anc
delta: {delta}
stage:
  op: for_all
  src: N0.in_neigh
  dst_var: S
  skip_if: S == N1
stage:
  op: intersect
  src: S.out_neigh, N1.in_neigh
  dst_var: M
  skip_if: e1.amount > 300
emit:
  mode: source_count
  target: M
""",
    "union_sets": """pattern: union_sets
delta: {delta}
stage:
  op: for_all
  src: N0.in_neigh
  dst_var: A
stage:
  op: for_all
  src: N1.out_neigh
  dst_var: B
stage:
  op: union
  src: A.self, B.self
  dst_var: U
  skip_if: U == N0
  skip_if: U == N1
emit:
  mode: set_cardinality
  min_size: 2
  target: U
""",
    "set_adj": """pattern: set_adj
delta: {delta}
stage:
  op: for_all
  src: N0.in_neigh
  dst_var: A
stage:
  op: intersect
  src: A.self, N1.out_neigh
  dst_var: X
emit:
  mode: set_cardinality
  target: X
""",
    "sibling_ref": """pattern: sibling_ref
delta: {delta}
stage:
  op: for_all
  src: N0.in_neigh
  dst_var: P
stage:
  op: for_all
  src: N1.out_neigh
  dst_var: A
  skip_if: A == N0
stage:
  op: intersect
  src: A.out_neigh, P.self
  dst_var: Q
  order: e3.t < e2.t
emit:
  mode: set_cardinality
  target: Q
""",
    "fwd_order": """pattern: fwd_order
delta: {delta}
stage:
  op: for_all
  src: N1.out_neigh
  dst_var: A
  window: forward
  skip_if: A == N0
stage:
  op: intersect
  src: A.out_neigh, N0.in_neigh
  dst_var: C
  window: forward
  order: e2.t >= e1.t
  order: e3.t > t
emit:
  mode: source_count
  min_size: 1
  target: C
""",
    "amt_edges": """pattern: amt_edges
delta: {delta}
stage:
  op: for_all
  src: N0.in_neigh
  dst_var: I
  skip_if: e1.amount >= 250.5
  skip_if: e1.currency == "EUR"
stage:
  op: for_all
  src: I.in_neigh
  dst_var: J
  skip_if: J == N0
  skip_if: e2.amount < e1.amount
emit:
  mode: edge_count
  min_size: 2
  target: J
""",
}
VM_CUSTOMS = ("spray_union", "filtered_senders", "sg_ordered", "stack_forward", "chain_5cycle")
VM_VOCAB = ("USD", "EUR", "GBP", "CHF")


def vm_texts(delta: int, attribution: str = "trigger") -> dict:
    import re
    out = {}
    for name in VM_CUSTOMS:
        txt = (CUSTOM_DIR / f"{name}.pat").read_text()
        out[name] = re.sub(r"(?m)^delta:.*$", f"delta: {delta}", txt)
    for name, tmpl in VM_PATTERNS.items():
        out[name] = tmpl.replace("{delta}", str(delta))
    if attribution != "trigger":
        out = {n: re.sub(r"(?m)^(delta:.*)$", rf"\1\nattribution: {attribution}", t) for n, t in out.items()}
    return out


def vm_plans(delta: int, attribution: str = "trigger"):
    return [compile_pattern(dsl.must_validate(dsl.parse_pattern(t)), None, force_generic=True)
            for t in vm_texts(delta, attribution).values()]


def vm_graph(edges):
    """edges (src, dst, t) with deterministic amounts / currencies."""
    recs = [TransactionRecord(i, int(e[0]), int(e[1]), int(e[2]), float(50 + (i * 37) % 1000),
                              VM_VOCAB[(i * 3 + i // 5) % 4]) for i, e in enumerate(edges)]
    return build_graph(recs)


def vm_case(edges, delta, want_instances):
    g = vm_graph(edges)
    plans = vm_plans(delta)
    fm = mine(g, plans)
    counts = np.stack([fm.column(p.name) for p in plans], axis=1)
    fmm = mine(g, vm_plans(delta, "members"))
    members = np.stack([fmm.column(p.name) for p in plans], axis=1)
    rec = np.zeros(0, dtype=np.int32)
    if want_instances:
        _, inst = mine(g, plans, collect_instances=True)
        col = {p.name: i for i, p in enumerate(plans)}
        out = []
        for r in inst:
            out += [col[r.pattern], r.trigger_edge, len(r.member_edges), len(r.member_nodes)]
            out += list(r.member_edges) + list(r.member_nodes)
        rec = np.array(out, dtype=np.int32)
    return (np.asarray(edges, dtype=np.int64).reshape(-1, 3), g.edge_amount.copy(),
            g.edge_currency.copy(), tuple(g.currency_vocab), counts, members, rec)


def _vm_one(args):
    return vm_case(*args)


VM_CORPUS = 40


def make_vm():
    vm_plans(0), vm_plans(5, "members")  # validate every program up front
    jobs, meta = [], []
    for name, (edges, deltas) in HAND_GRAPHS.items():
        for d in deltas:
            jobs.append((edges, d, True))
            meta.append({"name": name, "delta": d})
    for i, p in enumerate(corpus_params()[:VM_CORPUS]):
        seed, n_nodes, n_edges, horizon, deltas = p
        edges = corpus_records(seed, n_nodes, n_edges, horizon)
        for k, d in enumerate(deltas):
            jobs.append((edges, int(d), k == 0 and i < 24))
            meta.append({"name": f"corpus{i}", "delta": int(d)})
    z = np.load(OUT / "ties.npz")
    te = np.stack([z["src0"], z["dst0"], z["time0"]], axis=1).astype(np.int64)
    for d in (0, 2):
        jobs.append((te.tolist(), d, False))
        meta.append({"name": "ties0", "delta": d})
    t0 = time.time()
    with multiprocessing.get_context("fork").Pool(os.cpu_count()) as pool:
        res = pool.map(_vm_one, jobs, chunksize=1)
    arrays = {}
    for k, (edges, amount, cur, vocab, counts, members, rec) in enumerate(res):
        meta[k]["vocab"] = list(vocab)
        arrays[f"edges{k}"] = edges
        arrays[f"amount{k}"] = amount
        arrays[f"currency{k}"] = cur
        arrays[f"counts{k}"] = counts
        arrays[f"members{k}"] = members
        arrays[f"rec{k}"] = rec
    plans = [dataclasses.asdict(p) for p in vm_plans(0)]
    np.savez_compressed(OUT / "vm.npz", meta=json.dumps(meta), plans=json.dumps(plans), **arrays)
    words = sum(len(r[-1]) for r in res)
    print(f"vm.npz: {len(meta)} cases, {len(plans)} programs, {words} record words, {time.time() - t0:.0f}s")


# ---------------------------------------------------------------------------
# VM predicates on timestamps beyond 2^53: the reference compares a Python
# int (edge time / id) with a float (amount, DSL number) exactly


BIGT_TEXT = """pattern: bigt
delta: {delta}
stage:
  op: for_all
  src: N0.in_neigh
  dst_var: A
  skip_if: e1.amount < e1.t
emit:
  mode: edge_count
  target: A
"""
BIGT_TEXT2 = """pattern: bigt_ge
delta: {delta}
stage:
  op: for_all
  src: N1.out_neigh
  dst_var: B
  skip_if: e1.amount >= e1.t
emit:
  mode: edge_count
  target: B
"""


def make_vm_bigtime():
    base = 1 << 60
    rng = random.Random(53)
    edges, amounts = [], []
    for i in range(400):
        s, d = rng.randrange(12), rng.randrange(12)
        t = base + rng.randrange(0, 64)
        edges.append((s, d, t))
        # amounts exactly representable near 2^60 (spacing 256): some equal a
        # time's double rounding but not the time itself
        amounts.append(float(base + 256 * rng.randrange(-1, 2)))
    recs = [TransactionRecord(i, e[0], e[1], e[2], amounts[i], "USD") for i, e in enumerate(edges)]
    g = build_graph(recs)
    out = {"edges": [list(map(int, e)) for e in edges], "amount": amounts, "cases": []}
    for delta in (0, 7, 64):
        plans = [compile_pattern(dsl.must_validate(dsl.parse_pattern(t.replace("{delta}", str(delta)))), None,
                                 force_generic=True) for t in (BIGT_TEXT, BIGT_TEXT2)]
        fm = mine(g, plans)
        out["cases"].append({"delta": delta, "plans": [dataclasses.asdict(p) for p in plans],
                             "counts": [fm.column(p.name).tolist() for p in plans]})
    (OUT / "vm_bigtime.json").write_text(json.dumps(out))
    print("vm_bigtime.json:", [sum(map(sum, c["counts"])) for c in out["cases"]])


if __name__ == "__main__":
    which = sys.argv[1:] or ["hand", "corpus", "ties", "cfg1"]
    for w in which:
        globals()[f"make_{w}"]()
