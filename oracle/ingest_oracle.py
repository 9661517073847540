"""CPU restatement of the reference's ingestion — TEST INFRASTRUCTURE ONLY.

Restates txgraph.parse_transactions (txgraph.py:253-314), _resolve_columns
(:207-234), _parse_timestamp (:237-247) and build_graph (:317-354) with
plain Python (csv.reader, int(), float(), datetime.strptime, dicts).  It is
the checker for the GPU parser (paper_2604_12241_b200.ingest) at sizes the
committed golden fixtures do not cover, and is itself pinned to the
reference's outputs by tests/test_ingest_host.py (tests/golden/ingest.npz).
Never imported by the product.
"""

from __future__ import annotations

import csv
import io
from datetime import datetime, timezone

import numpy as np


class OracleParseError(ValueError):
    def __init__(self, message, line=None):
        self.line = line
        super().__init__(f"line {line}: {message}" if line is not None else message)


class OracleMappingError(ValueError):
    pass


def resolve_columns(header, m: dict) -> dict:
    """txgraph.py:207-234"""
    positions: dict = {}
    for i, name in enumerate(header):
        positions.setdefault(name.strip(), []).append(i)
    used: dict = {}

    def col(name, field):
        if name is None:
            return None
        idxs = positions.get(name)
        if not idxs:
            raise OracleMappingError(f"column {name!r} (mapped as {field}) not found in header {list(header)!r}")
        k = used.get(name, 0)
        used[name] = k + 1
        return idxs[min(k, len(idxs) - 1)]

    return {f: col(m[f], f) for f in ("timestamp", "src_bank", "src_account", "dst_bank", "dst_account",
                                       "amount", "currency", "label")}


DEFAULTS = dict(timestamp="Timestamp", src_bank="From Bank", src_account="Account", dst_bank="To Bank",
                dst_account="Account", amount="Amount Paid", currency="Payment Currency", label="Is Laundering",
                timestamp_format="%Y/%m/%d %H:%M", tick_seconds=1, delimiter=",")


def parse(data: bytes, **mapping):
    """-> dict of build_graph arrays (src, dst, time, amount, currency, label),
    node_count, vocab; raises OracleParseError / OracleMappingError."""
    m = {**DEFAULTS, **mapping}
    reader = csv.reader(io.StringIO(data.decode("utf-8"), newline=""), delimiter=m["delimiter"])
    try:
        header = next(reader)
    except StopIteration:
        raise OracleParseError("empty input: missing header row", line=1) from None
    cols = resolve_columns(header, m)
    needed = max(i for i in cols.values() if i is not None)
    ids: dict = {}
    vocab: dict = {}

    def node(bi, ai, row):
        key = (row[bi].strip(), row[ai].strip()) if bi is not None else row[ai].strip()
        v = ids.get(key)
        if v is None:
            v = ids[key] = len(ids)
        return v

    src, dst, tim, amt, cur, lab = [], [], [], [], [], []
    for lineno, row in enumerate(reader, start=2):
        if not row or (len(row) == 1 and not row[0].strip()):
            continue
        if len(row) <= needed:
            raise OracleParseError(f"expected at least {needed + 1} columns, got {len(row)}", line=lineno)
        try:
            text = row[cols["timestamp"]].strip()
            try:
                ts = int(text)
            except ValueError:
                if m["timestamp_format"] is None:
                    raise ValueError(f"timestamp {text!r} is not an integer tick count") from None
                dt = datetime.strptime(text, m["timestamp_format"]).replace(tzinfo=timezone.utc)
                ts = int(dt.timestamp()) // max(m["tick_seconds"], 1)
            if ts < 0:
                raise ValueError(f"negative timestamp {ts}")
            a = float(row[cols["amount"]]) if cols["amount"] is not None else 0.0
        except ValueError as exc:
            raise OracleParseError(str(exc), line=lineno) from None
        c = row[cols["currency"]].strip() if cols["currency"] is not None else ""
        lb = -1
        if cols["label"] is not None:
            raw = row[cols["label"]].strip().lower()
            if raw in ("1", "true", "yes"):
                lb = 1
            elif raw in ("0", "false", "no", ""):
                lb = 0
            else:
                raise OracleParseError(f"unrecognized label value {raw!r}", line=lineno)
        src.append(node(cols["src_bank"], cols["src_account"], row))
        dst.append(node(cols["dst_bank"], cols["dst_account"], row))
        tim.append(ts)
        amt.append(a)
        code = vocab.get(c)
        if code is None:
            code = vocab[c] = len(vocab)
        cur.append(code)
        lab.append(lb)
    return {"src": np.array(src, np.int64), "dst": np.array(dst, np.int64), "time": np.array(tim, np.int64),
            "amount": np.array(amt, np.float64), "currency": np.array(cur, np.int32),
            "label": np.array(lab, np.int8), "node_count": len(ids), "vocab": list(vocab)}
