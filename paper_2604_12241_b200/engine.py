"""`mine` — the drop-in replacement of tempmine.engine.mine (engine.py:658-712).

Same signature, same column order (order_plans, engine.py:596-604), same
errors (EngineInvariantError for duplicate names / slot mismatch, ValueError
for workers < 1), same return type (FeatureMatrix, engine.py:55-103).  The
work runs in libtempmine_b200.so on one GPU; `workers` is accepted for API
compatibility (the reference's fork-pool width) and has no effect — the
whole trigger range is one launch, balanced on the device.  Columns with
attribution "members" go through tm_mine_members (full-matrix
contributions, engine.py:629-640).  GENERIC plans that match no GPU family
run on the device stage VM (vm.py, csrc/tm_vm.cu — the reference's generic
interpreter, engine.py:325-562).  collect_instances=True returns the
reference's (FeatureMatrix, [InstanceRecord]) pair.  What neither path can
express raises UnsupportedPlanError instead of silently falling back to a
CPU interpreter.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib, hostmem
from .graph import DeviceGraph, as_device_graph
from .plan import BUILTIN_COLUMNS, GENERIC, PlanDesc, lower_plan
from .vm import VmProgram, lower_program, vm_instance_stream, vm_members, vm_mine


class EngineInvariantError(RuntimeError):
    """engine.py:33"""


@dataclass
class FeatureMatrix:
    """Per-edge pattern counts plus the edge identity columns (engine.py:55-103)."""

    columns: tuple
    values: np.ndarray  # (edge_count, len(columns)) int64
    edge_src: np.ndarray
    edge_dst: np.ndarray
    edge_time: np.ndarray
    edge_label: np.ndarray
    # the device graph these rows were mined on: to_csv formats on the GPU
    device_graph: object = field(default=None, repr=False, compare=False)

    @property
    def edge_count(self) -> int:
        return len(self.edge_src)

    def column(self, name: str) -> np.ndarray:
        return self.values[:, self.columns.index(name)]

    def to_csv(self, path: str) -> None:
        """edge_id,src,dst,timestamp,label,<features> — byte-identical to the
        reference writer (engine.py:73-103): empty label cell when < 0.
        Rows are formatted on the GPU (tm_csv_format) when the matrix came
        from a device graph, else on the host."""
        if self.device_graph is not None:
            return self._to_csv_gpu(path)
        n = self.edge_count
        with open(path, "w", encoding="utf-8", newline="\n") as fh:
            fh.write("edge_id,src,dst,timestamp,label")
            for col in self.columns:
                fh.write("," + col)
            fh.write("\n")
            chunk = 65536
            lab = np.asarray(self.edge_label).astype(np.int64)
            for start in range(0, n, chunk):
                stop = min(start + chunk, n)
                ids = np.arange(start, stop, dtype=np.int64).astype(str)
                cols = [ids, np.asarray(self.edge_src[start:stop], dtype=np.int64).astype(str),
                        np.asarray(self.edge_dst[start:stop], dtype=np.int64).astype(str),
                        np.asarray(self.edge_time[start:stop], dtype=np.int64).astype(str)]
                lab_s = lab[start:stop].astype(str)
                lab_s[lab[start:stop] < 0] = ""
                cols.append(lab_s)
                for j in range(len(self.columns)):
                    cols.append(self.values[start:stop, j].astype(str))
                rows = cols[0]
                for c in cols[1:]:
                    rows = np.char.add(np.char.add(rows, ","), c)
                fh.write("\n".join(rows.tolist()))
                fh.write("\n")


    def _to_csv_gpu(self, path: str) -> None:
        dg = self.device_graph
        vals = np.ascontiguousarray(self.values, dtype=np.int64)
        if vals.shape != (dg.edge_count, len(self.columns)):
            raise ValueError("values do not match the device graph")
        lab = np.ascontiguousarray(self.edge_label, dtype=np.int8)
        n = ctypes.c_int64()
        lib = _lib.load()
        with dg.lock:  # format + fetch share the graph's text buffer: one unit
            _lib.check(lib.tm_csv_format(dg.handle, _lib.ptr(vals), 0, vals.shape[1], _lib.ptr(lab),
                                         ctypes.byref(n)), "tm_csv_format")
            buf = np.empty(n.value, dtype=np.uint8)
            _lib.check(lib.tm_csv_fetch(dg.handle, _lib.ptr(buf), n.value), "tm_csv_fetch")
        with open(path, "wb") as fh:
            fh.write(("edge_id,src,dst,timestamp,label" + "".join("," + c for c in self.columns)
                      + "\n").encode("utf-8"))
            fh.write(memoryview(buf))


@dataclass(frozen=True)
class InstanceRecord:
    """One concrete matched instance (member_edges includes the trigger),
    engine.py:37-52."""

    pattern: str
    trigger_edge: int
    member_edges: tuple
    member_nodes: tuple

    def to_json_dict(self) -> dict:
        return {
            "pattern": self.pattern,
            "trigger_edge": self.trigger_edge,
            "member_edges": list(self.member_edges),
            "member_nodes": list(self.member_nodes),
        }


def merge_features(partials: list) -> FeatureMatrix:
    """engine.py:106-120 — elementwise integer sum."""
    if not partials:
        raise EngineInvariantError("nothing to merge")
    first = partials[0]
    total = first.values.copy()
    for other in partials[1:]:
        if tuple(other.columns) != tuple(first.columns):
            raise EngineInvariantError(f"column mismatch in merge: {other.columns} vs {first.columns}")
        if other.values.shape != first.values.shape:
            raise EngineInvariantError("row-count mismatch in merge")
        total += other.values
    return FeatureMatrix(first.columns, total, first.edge_src, first.edge_dst, first.edge_time,
                         first.edge_label)


def order_plans(plans: list) -> list:
    """engine.py:596-604 — builtin columns first in canonical order, then the
    rest in the order given; duplicate names are an error."""
    names = [p.name for p in plans]
    if len(set(names)) != len(names):
        raise EngineInvariantError(f"duplicate pattern names in {names}")
    builtin = [p for name in BUILTIN_COLUMNS for p in plans if p.name == name]
    custom = [p for p in plans if p.name not in BUILTIN_COLUMNS]
    return builtin + custom


def lower_all(plans: list, vocab=None, allow_vm: bool = False) -> tuple[list, list]:
    """Ordered plans and their lowering: a PlanDesc per family plan and, with
    allow_vm, a VmProgram per GENERIC plan no family matches."""
    plans = order_plans(list(plans))
    for p in plans:
        if p.slot_count != len(p.cells):
            raise EngineInvariantError(f"plan {p.name}: slot count disagrees with cells")
    items = []
    for p in plans:
        try:
            items.append(lower_plan(p))
        except _lib.UnsupportedPlanError:
            if not allow_vm or getattr(p, "kernel_hint", GENERIC) != GENERIC:
                raise
            items.append(lower_program(p, vocab))
    return plans, items


def _chunks(idx: list, n: int = _lib.MAX_PLANS):
    return [idx[i:i + n] for i in range(0, len(idx), n)]


def mine_members(dgraph: DeviceGraph, descs: list[PlanDesc], lo: int = 0, hi: int | None = None,
                 out: np.ndarray | None = None) -> np.ndarray:
    """Members attribution of triggers [lo, hi): full (n_edges, len(descs)) block
    (engine.py:629-640) — every counted instance adds 1 to each member row."""
    hi = dgraph.edge_count if hi is None else hi
    if out is None:
        out = np.empty((dgraph.edge_count, len(descs)), dtype=np.int64)
    if not descs or dgraph.edge_count == 0:
        out[:] = 0
        return out
    arr = _lib.plan_array(descs)
    with dgraph.lock:
        rc = _lib.load().tm_mine_members(dgraph.handle, arr, len(descs), lo, hi, _lib.ptr(out), 0, None)
        _lib.check(rc, "tm_mine_members")
    return out


def mine_rows(dgraph: DeviceGraph, descs: list[PlanDesc], lo: int, hi: int,
              out: np.ndarray | None = None) -> np.ndarray:
    """Rows [lo, hi) x len(descs) into a host int64 array (C order)."""
    rows = hi - lo
    if any(d.members for d in descs):
        raise ValueError("mine_rows takes trigger-attribution columns; use mine_members")
    if out is None:
        out = np.empty((rows, len(descs)), dtype=np.int64)
    if rows == 0 or not descs:
        return out
    arr = _lib.plan_array(descs)
    with dgraph.lock:
        rc = _lib.load().tm_mine(dgraph.handle, arr, len(descs), lo, hi, _lib.ptr(out), 0, None)
        _lib.check(rc, "tm_mine")
    return out


def mine_rows_device(dgraph: DeviceGraph, descs: list[PlanDesc], lo: int, hi: int, out_ptr: int,
                     stream: int | None = None) -> None:
    """Enqueue rows [lo, hi) into a device int64 buffer at out_ptr (row-major,
    len(descs) columns) on `stream`; returns without synchronizing."""
    if any(d.members for d in descs):
        raise ValueError("mine_rows_device takes trigger-attribution columns; use mine_members_device")
    if hi <= lo or not descs:
        return
    arr = _lib.plan_array(descs)
    with dgraph.lock:
        rc = _lib.load().tm_mine(dgraph.handle, arr, len(descs), lo, hi, ctypes.c_void_p(out_ptr), 1,
                                 ctypes.c_void_p(stream) if stream else None)
        _lib.check(rc, "tm_mine")


def prepare_views(dgraph: DeviceGraph, descs: list[PlanDesc], lo: int, hi: int, stream: int | None = None) -> None:
    """Build the window-start tables and time-slab views of `descs`' deltas for
    triggers [lo, hi) once (tm_mine_prepare): later mining calls on sub-ranges
    reuse them — e.g. the pieces of one multi-GPU step."""
    arr = _lib.plan_array([d for d in descs if isinstance(d, PlanDesc)])
    with dgraph.lock:
        _lib.check(_lib.load().tm_mine_prepare(dgraph.handle, arr, len(arr), lo, hi,
                                               ctypes.c_void_p(stream) if stream else None), "tm_mine_prepare")


def release_views(dgraph: DeviceGraph) -> None:
    """Forget the tables of prepare_views (tm_mine_release)."""
    with dgraph.lock:
        _lib.check(_lib.load().tm_mine_release(dgraph.handle), "tm_mine_release")


def mine_members_device(dgraph: DeviceGraph, descs: list[PlanDesc], lo: int, hi: int, out_ptr: int,
                        stream: int | None = None) -> None:
    """Enqueue members attribution of triggers [lo, hi): contributions are
    ADDED into the full (n_edges, len(descs)) device block at out_ptr — a
    sum over trigger ranges, so ranks combine with an all-reduce."""
    if hi <= lo or not descs:
        return
    arr = _lib.plan_array(descs)
    with dgraph.lock:
        rc = _lib.load().tm_mine_members(dgraph.handle, arr, len(descs), lo, hi, ctypes.c_void_p(out_ptr), 1,
                                         ctypes.c_void_p(stream) if stream else None)
        _lib.check(rc, "tm_mine_members")


# triggers per tm_collect_instances call: bounds the device record stream
INSTANCE_CHUNK = 1 << 16


def instance_stream(dgraph: DeviceGraph, descs: list[PlanDesc], lo: int, hi: int) -> np.ndarray:
    """Raw int32 record stream of triggers [lo, hi) (tempmine_b200.h:
    [plan, trigger, n_edges, n_nodes, edges..., nodes...] per record)."""
    if hi <= lo or not descs:
        return np.zeros(0, dtype=np.int32)
    lib = _lib.load()
    arr = _lib.plan_array(descs)
    words = ctypes.c_int64()
    with dgraph.lock:  # collect + fetch share the graph's record buffer: one unit
        _lib.check(lib.tm_collect_instances(dgraph.handle, arr, len(descs), lo, hi, ctypes.byref(words)),
                   "tm_collect_instances")
        buf = np.empty(words.value, dtype=np.int32)
        _lib.check(lib.tm_fetch_instances(dgraph.handle, _lib.ptr(buf), words.value), "tm_fetch_instances")
    return buf


def decode_instances(buf: np.ndarray, names: list) -> list:
    """Records -> InstanceRecord with member sets deduplicated and sorted
    (tuple(sorted(frozenset)), engine.py:641-645)."""
    out = []
    n = len(buf)
    p = 0
    data = buf.tolist()
    while p < n:
        ci, trig, ne, nn = data[p], data[p + 1], data[p + 2], data[p + 3]
        q = p + 4 + ne
        out.append(InstanceRecord(names[ci], trig, tuple(sorted(set(data[p + 4:q]))),
                                  tuple(sorted(set(data[q:q + nn])))))
        p = q + nn
    if p != n:
        raise EngineInvariantError("truncated instance stream")
    return out


def collect_instance_records(dgraph: DeviceGraph, descs: list[PlanDesc], names: list, lo: int = 0,
                             hi: int | None = None, sort: bool = True) -> list:
    """Every instance found at triggers [lo, hi), sorted like mine()'s
    (pattern, trigger_edge, member_edges) (engine.py:710-711)."""
    hi = dgraph.edge_count if hi is None else hi
    recs = []
    for a in range(lo, hi, INSTANCE_CHUNK):
        recs += decode_instances(instance_stream(dgraph, descs, a, min(a + INSTANCE_CHUNK, hi)), names)
    if sort:
        recs.sort(key=lambda r: (r.pattern, r.trigger_edge, r.member_edges))
    return recs


def last_stats(dgraph: DeviceGraph) -> _lib.TmMineStats:
    st = _lib.TmMineStats()
    with dgraph.lock:
        _lib.check(_lib.load().tm_last_mine_stats(dgraph.handle, ctypes.byref(st)), "tm_last_mine_stats")
    return st


def mine(graph, plans, workers: int = 1, collect_instances: bool = False, *, device: int = 0):
    """Mine every plan over every trigger edge on the GPU (engine.py:658).

    `graph` is a DeviceGraph or any TemporalGraph-like object (edge_src,
    edge_dst, edge_time, node_count); the latter is uploaded and built on the
    device once and cached for the lifetime of the graph object.
    """
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    vocab = getattr(graph, "currency_vocab", None)
    plans, items = lower_all(plans, vocab, allow_vm=True)
    dg = as_device_graph(graph, device)
    E = dg.edge_count
    # page-locked values: tm_mine overlaps its D2H with mining (hostmem.py)
    values = hostmem.pinned_empty((E, len(items)), np.int64)
    trig = [i for i, d in enumerate(items) if isinstance(d, PlanDesc) and not d.members]
    memb = [i for i, d in enumerate(items) if isinstance(d, PlanDesc) and d.members]
    if len(trig) == len(items) and len(items) <= _lib.MAX_PLANS:
        # the common case: every column in one launch, written in place
        mine_rows(dg, items, 0, E, out=values)
        trig = []
    for part in _chunks(trig):
        values[:, part] = mine_rows(dg, [items[i] for i in part], 0, E)
    for part in _chunks(memb):
        values[:, part] = mine_members(dg, [items[i] for i in part])
    for i, d in enumerate(items):
        if isinstance(d, VmProgram):
            values[:, i] = vm_members(dg, d) if d.members else vm_mine(dg, d)
    label = getattr(graph, "edge_label", None)
    if label is None:
        label = dg.edge_label
    fm = FeatureMatrix(columns=tuple(p.name for p in plans), values=values,
                       edge_src=graph.edge_src, edge_dst=graph.edge_dst,
                       edge_time=graph.edge_time, edge_label=label, device_graph=dg)
    if not collect_instances:
        return fm
    names = [p.name for p in plans]
    fam = [i for i, d in enumerate(items) if isinstance(d, PlanDesc)]
    recs = []
    for part in _chunks(fam):
        recs += collect_instance_records(dg, [items[i] for i in part], [names[i] for i in part], sort=False)
    for i, d in enumerate(items):
        if isinstance(d, VmProgram):
            for a in range(0, E, INSTANCE_CHUNK):
                recs += decode_instances(vm_instance_stream(dg, d, 0, a, min(a + INSTANCE_CHUNK, E)), [names[i]])
    recs.sort(key=lambda r: (r.pattern, r.trigger_edge, r.member_edges))
    return fm, recs


def write_instances(path: str, instances: list) -> None:
    """JSONL as the reference CLI writes it (cli.py:163-167)."""
    import json
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        for inst in instances:
            fh.write(json.dumps(inst.to_json_dict(), separators=(",", ":")) + "\n")
