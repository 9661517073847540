"""GPU ingestion (csrc/tm_ingest.cu) against the reference's own
parse_transactions + build_graph outputs (tests/golden/ingest.npz) and,
at sizes no fixture covers, against the pinned CPU restatement
(oracle/ingest_oracle.py)."""

from __future__ import annotations

import json
import random

import numpy as np
import pytest

from conftest import load_npz
from oracle import ingest_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def I():
    from paper_2604_12241_b200 import _lib, ingest
    _lib.load()
    return ingest


@pytest.fixture(scope="module")
def fx():
    z = load_npz("ingest.npz")
    return z, json.loads(str(z["meta"]))


def _same(t, want: dict, name: str):
    assert t.node_count == want["node_count"], name
    assert list(t.currency_vocab) == want["vocab"], name
    for key, got in (("src", t.edge_src), ("dst", t.edge_dst), ("time", t.edge_time),
                     ("currency", t.edge_currency), ("label", t.edge_label)):
        assert np.array_equal(got, want[key]), (name, key)
    assert np.array_equal(t.edge_amount.view(np.uint64), want["amount_bits"]), name


def test_reference_fixtures(I, fx):
    z, meta = fx
    for k, case in enumerate(meta):
        data = bytes(z[f"csv{k}"])
        mapping = I.ColumnMapping(**case["mapping"])
        if "error" in case:
            with pytest.raises((I.ParseError, I.MappingError)) as err:
                I.read_transactions(data, mapping)
            assert type(err.value).__name__ == case["error"], case["name"]
            assert getattr(err.value, "line", None) == case["line"], case["name"]
            assert str(err.value) == case["message"], case["name"]
            continue
        t = I.read_transactions(data, mapping)
        want = {key: z[f"{key}{k}"] for key in ("src", "dst", "time", "currency", "label", "amount_bits")}
        _same(t, {**want, "node_count": case["node_count"], "vocab": case["vocab"]}, case["name"])


def test_parse_transactions_records(I, fx):
    z, meta = fx
    k = [m["name"] for m in meta].index("three_rows")
    recs = I.parse_transactions(bytes(z[f"csv{k}"]))
    assert len(recs) == 3
    assert sorted({r.src for r in recs} | {r.dst for r in recs}) == [0, 1]
    assert [r.edge_id for r in recs] == [0, 1, 2]
    assert recs[2].label is True
    assert recs[0].timestamp == 100 and recs[0].amount == 50.0
    g = I.build_graph(recs)
    assert g.node_count == 2 and g.edge_count == 3
    with pytest.raises(I.GraphConstructionError):
        I.build_graph([])


def _ibm_like(n_rows: int, seed: int) -> bytes:
    rng = random.Random(seed)
    cur = ["US Dollar", "Euro", "Yuan", "Bitcoin", "Rupee", "UK Pound", "Saudi Riyal"]
    out = ["Timestamp,From Bank,Account,To Bank,Account,Amount Received,Receiving Currency,Amount Paid,"
           "Payment Currency,Payment Format,Is Laundering"]
    n_acc = max(10, n_rows // 8)
    for i in range(n_rows):
        if i % 997 == 13:
            out.append("")  # blank rows keep line numbers moving
        a1 = f"{int(rng.paretovariate(1.2)) % n_acc:09X}"
        a2 = f"{rng.randrange(n_acc):09X}"
        ts = f"2022/{rng.randint(1, 12)}/{rng.randint(1, 28):02d} {rng.randint(0, 23):02d}:{rng.randint(0, 59):02d}"
        amt = repr(rng.uniform(0.01, 1e7)) if i % 3 else f"{rng.uniform(0.01, 1e5):.2f}"
        c = rng.choice(cur)
        out.append(f"{ts},{rng.randint(0, 300):03d},{a1},{rng.randint(0, 300):03d},{a2},{amt},{c},{amt},{c},"
                   f"ACH,{int(rng.random() < 0.001)}")
    return ("\r\n".join(out) + "\r\n").encode()


def test_large_log_matches_oracle(I):
    data = _ibm_like(200_000, 3)
    t = I.read_transactions(data)
    want = O.parse(data)
    assert t.edge_count == 200_000
    _same(t, {**want, "amount_bits": want["amount"].view(np.uint64)}, "ibm_like_200k")


def test_ingest_csv_builds_the_same_graph(I):
    import paper_2604_12241_b200 as tmb
    data = _ibm_like(30_000, 5)
    g = I.ingest_csv(data)
    t = I.read_transactions(data)
    assert np.array_equal(g.edge_src, t.edge_src) and np.array_equal(g.edge_time, t.edge_time)
    h = tmb.DeviceGraph(t.edge_src, t.edge_dst, t.edge_time, node_count=t.node_count)
    for d in ("out", "in"):
        for a, b in zip(g.export_csr(d), h.export_csr(d)):
            assert np.array_equal(a, b)
    descs = [tmb.lower_plan(p) for p in tmb.full_pattern_set(86400)]
    assert np.array_equal(tmb.mine_rows(g, descs, 0, g.edge_count), tmb.mine_rows(h, descs, 0, h.edge_count))


def test_cache_round_trip_with_reference_bytes(I, fx, tmp_path):
    z, meta = fx
    k = int(z["cache_case"])
    path = tmp_path / "ref.tmg"
    path.write_bytes(bytes(z["cache_bytes"]))
    g = I.load_graph(str(path))
    assert g.node_count == meta[k]["node_count"]
    assert np.array_equal(g.edge_src, z[f"src{k}"]) and np.array_equal(g.edge_label, z[f"label{k}"])
    assert list(g.currency_vocab) == meta[k]["vocab"]
    out = tmp_path / "ours.tmg"
    I.save_graph(g, str(out))
    assert out.read_bytes() == bytes(z["cache_bytes"])


def test_unsupported_inputs_fail_loudly(I):
    hdr = b"Timestamp,Account,Account,Amount\n"
    m = I.ColumnMapping(src_bank=None, dst_bank=None, amount="Amount", currency=None, label=None)
    with pytest.raises(I.TempmineError, match="GPU CSV parser"):
        I.read_transactions(hdr + b'1,"a,b",c,1\n', m)
    with pytest.raises(I.TempmineError, match="line 3"):
        I.read_transactions(hdr + b"1,a,b,1\n2,a,b,12345678901234567891\n", m)
    with pytest.raises(I.TempmineError, match="line 2"):
        I.read_transactions(hdr + b"1,a,b,1_0.5\n", m)
