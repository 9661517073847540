"""Ingestion host logic on CPU: the oracle restatement against the
reference's own outputs (tests/golden/ingest.npz, make_ingest_golden.py),
the strptime program compiler, header resolution and the cache writer."""

from __future__ import annotations

import json
import types

import numpy as np
import pytest

from conftest import load_npz
from oracle import ingest_oracle as O
from paper_2604_12241_b200 import ingest as I


@pytest.fixture(scope="module")
def fx():
    z = load_npz("ingest.npz")
    return z, json.loads(str(z["meta"]))


def test_oracle_matches_reference_fixtures(fx):
    z, meta = fx
    assert len(meta) >= 40
    for k, case in enumerate(meta):
        data = bytes(z[f"csv{k}"])
        if "error" in case:
            with pytest.raises((O.OracleParseError, O.OracleMappingError)) as err:
                O.parse(data, **case["mapping"])
            assert type(err.value).__name__.replace("Oracle", "") == case["error"], case["name"]
            assert getattr(err.value, "line", None) == case["line"], case["name"]
            assert str(err.value) == case["message"], case["name"]
            continue
        got = O.parse(data, **case["mapping"])
        assert got["node_count"] == case["node_count"], case["name"]
        assert got["vocab"] == case["vocab"], case["name"]
        for key in ("src", "dst", "time", "currency", "label"):
            assert np.array_equal(got[key], z[f"{key}{k}"]), (case["name"], key)
        assert np.array_equal(got["amount"].view(np.uint64), z[f"amount_bits{k}"]), case["name"]


def test_timestamp_format_program():
    prog = I.compile_timestamp_format("%Y/%m/%d %H:%M")
    assert [op for op, _ in prog] == [I.F_Y, I.F_LIT, I.F_m, I.F_LIT, I.F_d, I.F_SPACE, I.F_H, I.F_LIT, I.F_M]
    assert prog[1] == (I.F_LIT, ord("/"))
    assert I.compile_timestamp_format(None) == []
    assert I.compile_timestamp_format("%%%S\t  %y") == [(I.F_LIT, 37), (I.F_S, 0), (I.F_SPACE, 0), (I.F_y, 0)]
    with pytest.raises(I.TempmineError, match="%b"):
        I.compile_timestamp_format("%d %b %Y")


def test_resolve_columns_positional_duplicates():
    hdr = "Timestamp,From Bank,Account,To Bank,Account,Amount Paid,Payment Currency,Is Laundering".split(",")
    cols = I._resolve_columns(hdr, I.ColumnMapping())
    assert cols["src_account"] == 2 and cols["dst_account"] == 4
    with pytest.raises(I.MappingError, match="Zeitstempel"):
        I._resolve_columns(hdr, I.ColumnMapping(timestamp="Zeitstempel"))


def test_split_header_terminators():
    assert I._split_header(b"") == (None, 0)
    assert I._split_header(b"a,b\r\n1,2\n") == (["a", "b"], 5)
    assert I._split_header(b"a,b\r1,2") == (["a", "b"], 4)
    assert I._split_header(b"a,b") == (["a", "b"], 3)


def test_mapping_struct_layout():
    cols = I._resolve_columns("Timestamp,Account,Account".split(","),
                              I.ColumnMapping(src_bank=None, dst_bank=None, amount=None, currency=None, label=None))
    m = I._mapping_struct(cols, I.ColumnMapping(src_bank=None, dst_bank=None, amount=None, currency=None,
                                                label=None, timestamp_format=None))
    assert (m.col_timestamp, m.col_src_account, m.col_dst_account, m.col_src_bank, m.needed) == (0, 1, 2, -1, 2)
    assert m.n_fmt == 0 and m.delimiter == ord(",")
    with pytest.raises(I.TempmineError, match="delimiter"):
        I._mapping_struct(cols, I.ColumnMapping(delimiter="ab"))


def test_save_graph_matches_reference_cache_bytes(fx, tmp_path):
    z, meta = fx
    k = int(z["cache_case"])
    want = bytes(z["cache_bytes"])
    g = types.SimpleNamespace(node_count=meta[k]["node_count"], edge_count=meta[k]["n_edges"],
                              edge_src=z[f"src{k}"], edge_dst=z[f"dst{k}"], edge_time=z[f"time{k}"],
                              edge_amount=z[f"amount_bits{k}"].view(np.float64), edge_currency=z[f"currency{k}"],
                              edge_label=z[f"label{k}"], currency_vocab=tuple(meta[k]["vocab"]))
    path = tmp_path / "g.tmg"
    I.save_graph(g, str(path))
    assert path.read_bytes() == want


def test_cache_errors(tmp_path):
    bad = tmp_path / "bad.tmg"
    bad.write_bytes(b"NOTCACHE" + bytes(32))
    with pytest.raises(I.CacheFormatError, match="magic"):
        I.load_graph(str(bad))
    ver = tmp_path / "ver.tmg"
    import struct
    ver.write_bytes(I.MAGIC + struct.pack("<IIQQII", 2, 0, 1, 1, 0, 0))
    with pytest.raises(I.CacheFormatError, match="version"):
        I.load_graph(str(ver))
    tr = tmp_path / "tr.tmg"
    tr.write_bytes(I.MAGIC + struct.pack("<IIQQII", 1, 0, 4, 100, 0, 0) + bytes(64))
    with pytest.raises(I.CacheFormatError, match="truncated"):
        I.load_graph(str(tr))
