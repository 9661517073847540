"""Transaction-log ingestion on the GPU.

Host mirror of the reference's ingestion API (txgraph.py:20-72, 207-354,
cache.py:40-81) over the C ABI's tm_ingest_* (csrc/tm_ingest.cu):

* `ColumnMapping`, `TransactionRecord`, `ParseError`, `MappingError`,
  `GraphConstructionError` — same fields, defaults and exception types.
* `read_transactions(source, mapping)` — the GPU parse: an `EdgeTable` of
  build_graph-shaped numpy arrays (src, dst, time, amount, currency, label,
  currency_vocab) with first-seen dense node ids.
* `parse_transactions(source, mapping)` -> list[TransactionRecord] and
  `build_graph(records)` -> DeviceGraph: the reference's two-step API.
* `ingest_csv(source, mapping)` -> DeviceGraph: the fused fast path — the
  parsed edge arrays never leave the device before the CSR build.
* `save_graph` / `load_graph`: the reference's versioned cache format v1.

Only the header row is read on the host (`_resolve_columns`, the same
positional duplicate-name rule as txgraph.py:207-234).  Row errors are found
on the GPU; the host re-reads the ONE failing row to word the ParseError
exactly like the reference (line numbers count csv rows, header = line 1).
"""

from __future__ import annotations

import csv
import ctypes
import io
import os
import struct
from dataclasses import dataclass
from datetime import datetime, timezone
from typing import IO, Iterable, Sequence

import numpy as np

from . import _lib
from ._lib import TempmineError
from .graph import DeviceGraph

# enum tm_parse_status / tm_fmt_op (include/tempmine_b200.h)
P_OK, P_COLUMNS, P_TIMESTAMP, P_NEGATIVE, P_AMOUNT, P_LABEL, P_UNSUPPORTED, P_COLLISION = range(8)
F_END, F_LIT, F_SPACE, F_Y, F_y, F_m, F_d, F_H, F_M, F_S = range(10)
_DIRECTIVES = {"Y": F_Y, "y": F_y, "m": F_m, "d": F_d, "H": F_H, "M": F_M, "S": F_S}


class ParseError(ValueError):
    """Malformed input row. `line` is 1-based (header is line 1). txgraph.py:20-28"""

    def __init__(self, message: str, line: int | None = None):
        self.line = line
        if line is not None:
            message = f"line {line}: {message}"
        super().__init__(message)


class MappingError(ValueError):
    """A ColumnMapping names a column the header does not have. txgraph.py:31-32"""


class GraphConstructionError(ValueError):
    """Records violate a TemporalGraph precondition. txgraph.py:35-36"""


@dataclass(frozen=True, slots=True)
class TransactionRecord:
    """txgraph.py:39-47"""

    edge_id: int
    src: int
    dst: int
    timestamp: int
    amount: float
    currency: str
    label: bool | None = None


@dataclass(frozen=True)
class ColumnMapping:
    """txgraph.py:50-72 — defaults match the IBM AML CSV layout."""

    timestamp: str = "Timestamp"
    src_bank: str | None = "From Bank"
    src_account: str = "Account"
    dst_bank: str | None = "To Bank"
    dst_account: str = "Account"
    amount: str | None = "Amount Paid"
    currency: str | None = "Payment Currency"
    label: str | None = "Is Laundering"
    timestamp_format: str | None = "%Y/%m/%d %H:%M"
    tick_seconds: int = 1
    delimiter: str = ","


@dataclass
class EdgeTable:
    """build_graph's arrays (txgraph.py:330-354) plus the row count."""

    node_count: int
    edge_src: np.ndarray
    edge_dst: np.ndarray
    edge_time: np.ndarray
    edge_amount: np.ndarray
    edge_currency: np.ndarray
    edge_label: np.ndarray
    currency_vocab: tuple
    n_rows: int

    @property
    def edge_count(self) -> int:
        return len(self.edge_src)


def _resolve_columns(header: Sequence[str], mapping: ColumnMapping) -> dict:
    """txgraph.py:207-234: duplicate header names are consumed positionally."""
    positions: dict[str, list[int]] = {}
    for i, name in enumerate(header):
        positions.setdefault(name.strip(), []).append(i)
    used: dict[str, int] = {}

    def col(name, field):
        if name is None:
            return None
        idxs = positions.get(name)
        if not idxs:
            raise MappingError(f"column {name!r} (mapped as {field}) not found in header {list(header)!r}")
        k = used.get(name, 0)
        used[name] = k + 1
        return idxs[min(k, len(idxs) - 1)]

    return {
        "timestamp": col(mapping.timestamp, "timestamp"),
        "src_bank": col(mapping.src_bank, "src_bank"),
        "src_account": col(mapping.src_account, "src_account"),
        "dst_bank": col(mapping.dst_bank, "dst_bank"),
        "dst_account": col(mapping.dst_account, "dst_account"),
        "amount": col(mapping.amount, "amount"),
        "currency": col(mapping.currency, "currency"),
        "label": col(mapping.label, "label"),
    }


def compile_timestamp_format(fmt: str | None) -> list[tuple[int, int]]:
    """ColumnMapping.timestamp_format -> device strptime program.

    Mirrors _strptime.TimeRE.pattern: whitespace runs become \\s+, '%%' a
    literal '%', other characters literals (matched case-insensitively);
    directives Y y m d H M S.  Anything else is outside the GPU parser."""
    if fmt is None:
        return []
    ops: list[tuple[int, int]] = []
    i = 0
    while i < len(fmt):
        c = fmt[i]
        if c == "%":
            if i + 1 >= len(fmt):
                raise TempmineError(_lib.TM_E_UNSUPPORTED_PLAN, f"timestamp_format {fmt!r}: trailing '%'")
            d = fmt[i + 1]
            if d == "%":
                ops.append((F_LIT, ord("%")))
            elif d in _DIRECTIVES:
                ops.append((_DIRECTIVES[d], 0))
            else:
                raise TempmineError(_lib.TM_E_UNSUPPORTED_PLAN,
                                    f"timestamp_format directive %{d} is not supported by the GPU parser")
            i += 2
        elif c.isspace():
            while i < len(fmt) and fmt[i].isspace():
                i += 1
            ops.append((F_SPACE, 0))
        else:
            if ord(c) > 127:
                raise TempmineError(_lib.TM_E_UNSUPPORTED_PLAN, f"timestamp_format {fmt!r}: non-ASCII literal")
            ops.append((F_LIT, ord(c)))
            i += 1
    if len(ops) > _lib.TM_FMT_MAX:
        raise TempmineError(_lib.TM_E_UNSUPPORTED_PLAN, f"timestamp_format {fmt!r} is too long")
    return ops


def _read_source(source) -> bytes:
    if isinstance(source, (bytes, bytearray, memoryview)):
        return bytes(source)
    if isinstance(source, (str, os.PathLike)):
        with open(source, "rb") as fh:
            return fh.read()
    if hasattr(source, "read"):
        data = source.read()
        return data.encode("utf-8") if isinstance(data, str) else bytes(data)
    if isinstance(source, Iterable):  # lines, like csv.reader accepts
        return "".join(source).encode("utf-8")
    raise TypeError(f"unsupported source {type(source)!r}")


def _split_header(data: bytes, delimiter: str = ",") -> tuple[list[str] | None, int]:
    """First csv row and the offset of the data rows (csv.reader line rule)."""
    if not data:
        return None, 0
    n_pos = data.find(b"\n")
    r_pos = data.find(b"\r")
    ends = [p for p in (n_pos, r_pos) if p >= 0]
    if not ends:
        head, start = data, len(data)
    else:
        e = min(ends)
        head = data[:e]
        start = e + 2 if data[e:e + 2] == b"\r\n" else e + 1
    rows = list(csv.reader(io.StringIO(head.decode("utf-8"), newline=""), delimiter=delimiter))
    return (rows[0] if rows else []), start


def _mapping_struct(cols: dict, mapping: ColumnMapping) -> _lib.TmCsvMapping:
    if len(mapping.delimiter) != 1 or ord(mapping.delimiter) > 127 or mapping.delimiter in "\r\n\"":
        raise TempmineError(_lib.TM_E_UNSUPPORTED_PLAN,
                            f"delimiter {mapping.delimiter!r}: the GPU parser takes one ASCII byte")
    m = _lib.TmCsvMapping()
    for key in ("timestamp", "src_bank", "src_account", "dst_bank", "dst_account", "amount", "currency",
                "label"):
        setattr(m, f"col_{key}", -1 if cols[key] is None else cols[key])
    m.needed = max(i for i in cols.values() if i is not None)
    m.delimiter = ord(mapping.delimiter)
    m.tick_seconds = max(int(mapping.tick_seconds), 1)
    prog = compile_timestamp_format(mapping.timestamp_format)
    m.n_fmt = len(prog)
    for k, (op, arg) in enumerate(prog):
        m.fmt_op[k] = op
        m.fmt_arg[k] = arg
    return m


def _row_error(row_text: str, status: int, cols: dict, mapping: ColumnMapping, line: int) -> Exception:
    """Word the ParseError of the first failing row like txgraph.py:284-308."""
    row = row_text.split(mapping.delimiter)
    needed = max(i for i in cols.values() if i is not None)
    if status == P_COLUMNS:
        return ParseError(f"expected at least {needed + 1} columns, got {len(row)}", line=line)
    if status in (P_TIMESTAMP, P_NEGATIVE):
        text = row[cols["timestamp"]].strip()
        try:
            ts = int(text)
        except ValueError:
            if mapping.timestamp_format is None:
                return ParseError(f"timestamp {text!r} is not an integer tick count", line=line)
            try:
                dt = datetime.strptime(text, mapping.timestamp_format).replace(tzinfo=timezone.utc)
            except ValueError as exc:
                return ParseError(str(exc), line=line)
            ts = int(dt.timestamp()) // max(mapping.tick_seconds, 1)
        if ts < 0:
            return ParseError(f"negative timestamp {ts}", line=line)
    elif status == P_AMOUNT:
        try:
            float(row[cols["amount"]])
        except ValueError as exc:
            return ParseError(str(exc), line=line)
    elif status == P_LABEL:
        raw = row[cols["label"]].strip().lower()
        return ParseError(f"unrecognized label value {raw!r}", line=line)
    elif status == P_COLLISION:
        return TempmineError(_lib.TM_E_STATE, "64-bit key hash collision between distinct accounts")
    if status == P_UNSUPPORTED:
        return TempmineError(_lib.TM_E_UNSUPPORTED_PLAN,
                             f"line {line}: input outside the GPU CSV parser (quoted fields, amounts with "
                             "more than 19 significant digits or subnormal values, '_' digit separators, "
                             "or timestamps beyond int64)")
    return TempmineError(_lib.TM_E_STATE, f"line {line}: GPU parser status {status} not confirmed by the host")


class _Parsed:
    """Owns a tm_ingest handle."""

    def __init__(self, handle, info):
        self.h = handle
        self.info = info

    def __del__(self):
        if getattr(self, "h", None):
            _lib.load().tm_ingest_free(self.h)
            self.h = None


def _ingest(source, mapping: ColumnMapping | None, device: int, stream=None):
    mapping = mapping or ColumnMapping()
    data = _read_source(source)
    header, start = _split_header(data, mapping.delimiter)
    if header is None:
        raise ParseError("empty input: missing header row", line=1)
    cols = _resolve_columns(header, mapping)
    m = _mapping_struct(cols, mapping)
    body = np.frombuffer(data, dtype=np.uint8, offset=start) if start < len(data) else np.empty(0, np.uint8)
    lib = _lib.load()
    h = ctypes.c_void_p()
    info = _lib.TmIngestInfo()
    _lib.check(lib.tm_ingest_csv(device, body.ctypes.data if len(body) else None, len(body), 0, ctypes.byref(m),
                                 stream, ctypes.byref(h), ctypes.byref(info)), "tm_ingest_csv")
    if info.err_row >= 0:
        line = int(info.err_row) + 2
        text = data[start + info.err_begin:start + info.err_end].decode("utf-8")
        if text.endswith("\r"):
            text = text[:-1]
        raise _row_error(text, int(info.err_status), cols, mapping, line)
    return _Parsed(h, info), cols


def _fetch(p: _Parsed, cols: dict) -> EdgeTable:
    lib = _lib.load()
    E = int(p.info.n_edges)
    src = np.empty(E, np.int64)
    dst = np.empty(E, np.int64)
    tim = np.empty(E, np.int64)
    amt = np.empty(E, np.float64)
    cur = np.empty(E, np.int32)
    lab = np.empty(E, np.int8)
    _lib.check(lib.tm_ingest_fetch(p.h, _lib.ptr(src), _lib.ptr(dst), _lib.ptr(tim), _lib.ptr(amt),
                                   _lib.ptr(cur), _lib.ptr(lab)), "tm_ingest_fetch")
    nc = int(p.info.n_currency)
    off = np.zeros(nc + 1, np.int64)
    _lib.check(lib.tm_ingest_vocab(p.h, _lib.ptr(off), None, 0), "tm_ingest_vocab")
    raw = np.empty(max(int(off[-1]), 1), np.uint8)
    _lib.check(lib.tm_ingest_vocab(p.h, _lib.ptr(off), _lib.ptr(raw), len(raw)), "tm_ingest_vocab")
    blob = raw.tobytes()
    vocab = tuple(blob[off[i]:off[i + 1]].decode("utf-8") for i in range(nc))
    return EdgeTable(int(p.info.n_nodes), src, dst, tim, amt, cur, lab, vocab, int(p.info.n_rows))


def read_transactions(source, mapping: ColumnMapping | None = None, device: int = 0) -> EdgeTable:
    """Parse a delimited transaction log on the GPU into build_graph arrays."""
    p, cols = _ingest(source, mapping, device)
    return _fetch(p, cols)


def parse_transactions(source: str | os.PathLike | IO[str] | Iterable[str],
                       mapping: ColumnMapping | None = None, device: int = 0) -> list[TransactionRecord]:
    """txgraph.py:253-314 — dense first-seen node ids, edge ids in row order."""
    t = read_transactions(source, mapping, device)
    vocab = t.currency_vocab
    return [TransactionRecord(i, int(s), int(d), int(ts), float(a), vocab[c], None if lb < 0 else bool(lb))
            for i, (s, d, ts, a, c, lb) in enumerate(zip(t.edge_src.tolist(), t.edge_dst.tolist(),
                                                         t.edge_time.tolist(), t.edge_amount.tolist(),
                                                         t.edge_currency.tolist(), t.edge_label.tolist()))]


def build_graph(records: Sequence[TransactionRecord], device: int = 0) -> DeviceGraph:
    """txgraph.py:317-354: validate the records and build the device graph."""
    if not records:
        raise GraphConstructionError("no records: cannot build an empty graph")
    n = len(records)
    src = np.empty(n, np.int64)
    dst = np.empty(n, np.int64)
    tim = np.empty(n, np.int64)
    amt = np.empty(n, np.float64)
    lab = np.empty(n, np.int8)
    cur = np.empty(n, np.int32)
    vocab: dict[str, int] = {}
    for i, rec in enumerate(records):
        if rec.edge_id != i:
            raise GraphConstructionError(f"edge_id {rec.edge_id} at position {i}: ids must be contiguous from 0")
        if rec.src < 0 or rec.dst < 0:
            raise GraphConstructionError(f"edge {i}: negative node id")
        if rec.timestamp < 0:
            raise GraphConstructionError(f"edge {i}: negative timestamp")
        src[i], dst[i], tim[i], amt[i] = rec.src, rec.dst, rec.timestamp, rec.amount
        lab[i] = -1 if rec.label is None else int(rec.label)
        code = vocab.get(rec.currency)
        if code is None:
            code = vocab[rec.currency] = len(vocab)
        cur[i] = code
    node_count = int(max(src.max(), dst.max())) + 1
    return DeviceGraph(src, dst, tim, node_count=node_count, edge_label=lab, device=device, edge_amount=amt,
                       edge_currency=cur, currency_vocab=tuple(vocab))


def ingest_csv(source, mapping: ColumnMapping | None = None, device: int = 0) -> DeviceGraph:
    """parse_transactions + build_graph fused: parse on the GPU and build the
    dual CSR from the parsed device arrays (no host round trip of the edge
    table before the build)."""
    p, cols = _ingest(source, mapping, device)
    if p.info.n_edges == 0:
        raise GraphConstructionError("no records: cannot build an empty graph")
    gh = ctypes.c_void_p()
    _lib.check(_lib.load().tm_ingest_graph(p.h, ctypes.byref(gh)), "tm_ingest_graph")
    t = _fetch(p, cols)
    for a in (t.edge_src, t.edge_dst, t.edge_time, t.edge_amount, t.edge_currency, t.edge_label):
        a.flags.writeable = False
    return DeviceGraph._adopt(gh, t.node_count, t.edge_src, t.edge_dst, t.edge_time, t.edge_label,
                              t.edge_amount, t.edge_currency, t.currency_vocab, device)


# ------------------------------------------------------------------ cache v1

MAGIC = b"TMGCACHE"
VERSION = 1


class CacheFormatError(ValueError):
    """cache.py:37-38"""


def save_graph(graph, path: str) -> None:
    """cache.py:40-52 — byte-identical files for identical graphs."""
    vocab = getattr(graph, "currency_vocab", None) or ()
    E = graph.edge_count
    amount = getattr(graph, "edge_amount", None)
    currency = getattr(graph, "edge_currency", None)
    label = getattr(graph, "edge_label", None)
    arrays = (np.asarray(graph.edge_src, "<i8"), np.asarray(graph.edge_dst, "<i8"),
              np.asarray(graph.edge_time, "<i8"),
              np.asarray(amount if amount is not None else np.zeros(E), "<f8"),
              np.asarray(currency if currency is not None else np.zeros(E, np.int32), "<i4"),
              np.asarray(label if label is not None else np.full(E, -1, np.int8), "i1"))
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<IIQQII", VERSION, 0, graph.node_count, E, len(vocab), 0))
        for arr in arrays:
            fh.write(np.ascontiguousarray(arr).tobytes())
        for code in vocab:
            raw = code.encode("utf-8")
            fh.write(struct.pack("<I", len(raw)))
            fh.write(raw)


def load_graph(path: str, device: int = 0) -> DeviceGraph:
    """cache.py:55-81 — the CSR is rebuilt (on the GPU) from the edge table."""
    with open(path, "rb") as fh:
        magic = fh.read(8)
        if magic != MAGIC:
            raise CacheFormatError(f"not a graph cache (bad magic {magic!r})")
        version, _, node_count, edge_count, n_currency, _ = struct.unpack("<IIQQII", fh.read(32))
        if version != VERSION:
            raise CacheFormatError(f"unsupported cache version {version} (expected {VERSION})")

        def read_array(dtype: str, count: int) -> np.ndarray:
            dt = np.dtype(dtype)
            raw = fh.read(dt.itemsize * count)
            if len(raw) != dt.itemsize * count:
                raise CacheFormatError("truncated cache file")
            return np.frombuffer(raw, dtype=dt).copy()

        src = read_array("<i8", edge_count)
        dst = read_array("<i8", edge_count)
        tim = read_array("<i8", edge_count)
        amount = read_array("<f8", edge_count)
        currency = read_array("<i4", edge_count)
        label = read_array("i1", edge_count)
        vocab = []
        for _ in range(n_currency):
            (ln,) = struct.unpack("<I", fh.read(4))
            vocab.append(fh.read(ln).decode("utf-8"))
    return DeviceGraph(src, dst, tim, node_count=node_count, edge_label=label, device=device,
                       edge_amount=amount, edge_currency=currency, currency_vocab=tuple(vocab))
