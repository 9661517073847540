"""Device-resident temporal graph (the GPU counterpart of TemporalGraph).

Reference: txgraph.py:106-204.  The host keeps the edge table (read-only
numpy views, as the reference marks its arrays, txgraph.py:164-170); the
dual CSR, time ranks and pair index live in HBM behind a tm_graph handle and
are built there by radix sorts (csrc/tm_graph.cu).
"""

from __future__ import annotations

import ctypes
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass(frozen=True)
class GraphStats:
    """txgraph.py:77-84 — per-direction degree summary used by plan compilers."""

    mean_out_degree: float
    mean_in_degree: float
    p99_out_degree: float
    p99_in_degree: float


def _as_i64(a, name: str) -> np.ndarray:
    arr = np.ascontiguousarray(np.asarray(a), dtype=np.int64)
    if arr.ndim != 1:
        raise ValueError(f"{name} must be one-dimensional")
    return arr


class DeviceGraph:
    """Immutable dual-CSR temporal multigraph resident on one GPU.

    Construct from edge arrays (`DeviceGraph(src, dst, time)`) or from any
    object with the reference TemporalGraph's edge fields
    (`DeviceGraph.from_graph(g)`).  node_count defaults to max id + 1
    (build_graph, txgraph.py:353).
    """

    def __init__(self, edge_src, edge_dst, edge_time, node_count: int | None = None,
                 edge_label=None, device: int = 0, stream: int | None = None, edge_amount=None,
                 edge_currency=None, currency_vocab=None):
        lib = _lib.load()
        src = _as_i64(edge_src, "edge_src")
        dst = _as_i64(edge_dst, "edge_dst")
        tim = _as_i64(edge_time, "edge_time")
        if not (len(src) == len(dst) == len(tim)):
            raise ValueError("edge arrays differ in length")
        if node_count is None:
            node_count = int(max(src.max(), dst.max())) + 1 if len(src) else 0
        self.node_count = int(node_count)
        self.edge_count = len(src)
        self.device = int(device)
        self.edge_src, self.edge_dst, self.edge_time = src, dst, tim
        if edge_label is None:
            edge_label = np.full(self.edge_count, -1, dtype=np.int8)
        self.edge_label = np.asarray(edge_label)
        handle = ctypes.c_void_p()
        rc = lib.tm_graph_build(self.device, self.node_count, self.edge_count, _lib.ptr(src),
                                _lib.ptr(dst), _lib.ptr(tim), 0, stream, ctypes.byref(handle))
        _lib.check(rc, "tm_graph_build")
        self._h = handle
        self._finalizer = weakref.finalize(self, lib.tm_graph_free, handle)
        # every C call sequence on the handle runs under this lock: the calls
        # share the handle's scratch and result buffers (tempmine_b200.h)
        self.lock = threading.RLock()
        self._stats: GraphStats | None = None
        self._csr: dict = {}
        # edge attributes (txgraph.py:113-123), uploaded on first use by an
        # attribute predicate of a GENERIC stage program
        self.edge_amount = edge_amount
        self.edge_currency = edge_currency
        self.currency_vocab = tuple(currency_vocab) if currency_vocab is not None else None
        self._attrs_on_device = False

    def ensure_attrs(self) -> None:
        """Upload amount / currency / vocabulary ranks (tm_graph_set_attrs)."""
        if self._attrs_on_device:
            return
        if self.edge_amount is None or self.edge_currency is None or self.currency_vocab is None:
            raise ValueError("attribute predicates need edge_amount, edge_currency and currency_vocab")
        amount = np.ascontiguousarray(self.edge_amount, dtype=np.float64)
        cur = np.ascontiguousarray(self.edge_currency, dtype=np.int32)
        if len(amount) != self.edge_count or len(cur) != self.edge_count:
            raise ValueError("attribute arrays differ in length from the edge table")
        vocab = self.currency_vocab
        order = sorted(range(len(vocab)), key=lambda i: vocab[i])
        rank = np.empty(len(vocab), dtype=np.int32)
        rank[order] = np.arange(len(vocab), dtype=np.int32)
        with self.lock:
            _lib.check(_lib.load().tm_graph_set_attrs(self.handle, _lib.ptr(amount), _lib.ptr(cur),
                                                      len(vocab), _lib.ptr(rank)), "tm_graph_set_attrs")
        self._attrs_on_device = True

    @classmethod
    def _adopt(cls, handle: ctypes.c_void_p, node_count: int, edge_src, edge_dst, edge_time, edge_label,
               edge_amount, edge_currency, currency_vocab, device: int) -> "DeviceGraph":
        """Wrap a tm_graph built on the device (tm_ingest_graph): the host
        keeps read-only copies of the edge table like any other DeviceGraph."""
        self = cls.__new__(cls)
        self.node_count = int(node_count)
        self.edge_count = len(edge_src)
        self.device = int(device)
        self.edge_src, self.edge_dst, self.edge_time = edge_src, edge_dst, edge_time
        self.edge_label = edge_label
        self._h = handle
        self._finalizer = weakref.finalize(self, _lib.load().tm_graph_free, handle)
        self.lock = threading.RLock()
        self._stats = None
        self._csr = {}
        self.edge_amount = edge_amount
        self.edge_currency = edge_currency
        self.currency_vocab = tuple(currency_vocab) if currency_vocab is not None else None
        self._attrs_on_device = False
        return self

    @classmethod
    def from_graph(cls, graph, device: int = 0) -> "DeviceGraph":
        return cls(graph.edge_src, graph.edge_dst, graph.edge_time, node_count=graph.node_count,
                   edge_label=getattr(graph, "edge_label", None), device=device,
                   edge_amount=getattr(graph, "edge_amount", None),
                   edge_currency=getattr(graph, "edge_currency", None),
                   currency_vocab=getattr(graph, "currency_vocab", None))

    @property
    def handle(self) -> ctypes.c_void_p:
        if self._h is None:
            raise RuntimeError("graph was freed")
        return self._h

    def free(self) -> None:
        with self.lock:
            if self._h is not None:
                self._finalizer()
                self._h = None

    def info(self) -> _lib.TmGraphInfo:
        info = _lib.TmGraphInfo()
        with self.lock:
            _lib.check(_lib.load().tm_graph_info_get(self.handle, ctypes.byref(info)), "tm_graph_info_get")
        return info

    def degrees(self, direction: str) -> np.ndarray:
        out = np.empty(self.node_count, dtype=np.int64)
        d = 1 if direction == "out" else 0
        with self.lock:
            _lib.check(_lib.load().tm_graph_degrees(self.handle, d, _lib.ptr(out)), "tm_graph_degrees")
        return out

    @property
    def stats(self) -> GraphStats:
        """txgraph.py:155-162 (float summary; only orders intersect operands)."""
        if self._stats is None:
            do = self.degrees("out")
            di = self.degrees("in")
            if len(do) == 0:
                self._stats = GraphStats(0.0, 0.0, 0.0, 0.0)
            else:
                self._stats = GraphStats(float(do.mean()), float(di.mean()),
                                         float(np.percentile(do, 99)), float(np.percentile(di, 99)))
        return self._stats

    def export_csr(self, direction: str) -> tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
        """(indptr, nbr, time, eid) of the device CSR, as txgraph.py:137-144."""
        if direction not in self._csr:
            d = 1 if direction == "out" else 0
            n, e = self.node_count, self.edge_count
            indptr = np.empty(n + 1, dtype=np.int64)
            nbr = np.empty(e, dtype=np.int64)
            tim = np.empty(e, dtype=np.int64)
            eid = np.empty(e, dtype=np.int64)
            with self.lock:
                _lib.check(_lib.load().tm_graph_export_csr(self.handle, d, _lib.ptr(indptr), _lib.ptr(nbr),
                                                           _lib.ptr(tim), _lib.ptr(eid)),
                           "tm_graph_export_csr")
            for a in (indptr, nbr, tim, eid):
                a.flags.writeable = False
            self._csr[direction] = (indptr, nbr, tim, eid)
        return self._csr[direction]

    # reference-named views (txgraph.py:137-144)
    out_indptr = property(lambda self: self.export_csr("out")[0])
    out_nbr = property(lambda self: self.export_csr("out")[1])
    out_time = property(lambda self: self.export_csr("out")[2])
    out_eid = property(lambda self: self.export_csr("out")[3])
    in_indptr = property(lambda self: self.export_csr("in")[0])
    in_nbr = property(lambda self: self.export_csr("in")[1])
    in_time = property(lambda self: self.export_csr("in")[2])
    in_eid = property(lambda self: self.export_csr("in")[3])


_CACHE: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def as_device_graph(graph, device: int = 0) -> DeviceGraph:
    """DeviceGraph for `graph`, building (once per graph object) when given a
    host TemporalGraph-like object."""
    if isinstance(graph, DeviceGraph):
        return graph
    try:
        dg = _CACHE.get(graph)
    except TypeError:
        dg = None
    if dg is None or dg.device != device:
        dg = DeviceGraph.from_graph(graph, device=device)
        try:
            _CACHE[graph] = dg
        except TypeError:
            pass
    return dg
