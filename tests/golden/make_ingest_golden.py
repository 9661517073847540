"""Golden fixtures for GPU ingestion, produced by the REFERENCE itself.

Run in the build container only (the reference is mounted read-only at
/root/reference; it does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_ingest_golden.py

Each case is a CSV byte string plus a ColumnMapping; the expected result is
what `tempmine.txgraph.parse_transactions` + `build_graph`
(txgraph.py:253-354) return for it — the edge arrays, node count and
currency vocabulary — or the exception it raises (type, line, message).
Cases: the reference's own ingestion tests (test_txgraph.py:27-94, 205-209),
CSVs written by the reference's synth.write_csv (synth.py:166-178), and
edge cases of csv.reader / int() / float() / strptime / str.strip() the
GPU parser restates.  Writes tests/golden/ingest.npz.
"""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from tempmine import synth as rsynth  # noqa: E402
from tempmine.txgraph import ColumnMapping, build_graph, parse_transactions  # noqa: E402

OUT = Path(__file__).resolve().parent / "ingest.npz"
IBM = ("Timestamp,From Bank,Account,To Bank,Account,Amount Received,"
       "Receiving Currency,Amount Paid,Payment Currency,Payment Format,Is Laundering")


def ibm(rows, term="\n", trailing=True):
    text = term.join([IBM] + rows)
    return (text + (term if trailing else "")).encode("utf-8")


def cases():
    out = []

    def add(name, data, **mapping):
        out.append((name, data, mapping))

    # the reference's ingestion tests
    add("three_rows", ibm(["100,11,A1,11,A2,50,USD,50,USD,Wire,0", "101,11,A2,11,A1,60,USD,60,USD,Wire,0",
                           "102,11,A1,11,A2,70,USD,70,USD,Wire,1"]))
    add("datetime", ibm(["2022/09/01 00:20,1,X,2,Y,9.9,EUR,9.9,EUR,Wire,0"]))
    add("missing_columns", ibm(["100,1,A,2,B,5,USD,5,USD,Wire,0", "bad-row-without-enough-columns"]))
    add("bad_timestamp", ibm(["not-a-time,1,A,2,B,5,USD,5,USD,Wire,0"]))
    add("unknown_column", ibm(["100,1,A,2,B,5,USD,5,USD,Wire,0"]), timestamp="Zeitstempel")
    add("empty", b"")
    add("single_account", b"Timestamp,Account,Account,Amount Paid,Payment Currency\n5,alice,bob,1,USD\n",
        src_bank=None, dst_bank=None, label=None, amount="Amount Paid", currency="Payment Currency")
    add("first_seen", ibm(["10,9,zz,9,aa,1,USD,1,USD,Wire,0", "11,9,aa,9,bb,1,USD,1,USD,Wire,0"]))
    add("tick_seconds", ibm(["2022/09/01 00:20,1,X,2,Y,9.9,EUR,9.9,EUR,Wire,0"]), tick_seconds=60)
    # line terminators and blank rows (csv.reader)
    rows = ["5,1,A,1,B,1,USD,1,USD,Wire,0", "", "6,1,B,1,C,2,EUR,2,EUR,Wire,1", "   ",
            "7,2,A,1,A,3,USD,3,USD,Wire,0"]
    add("crlf", ibm(rows, "\r\n"))
    add("lone_cr", ibm(rows, "\r"))
    add("no_trailing_newline", ibm(rows, "\n", trailing=False))
    add("mixed_terms", (IBM + "\r\n" + rows[0] + "\n" + rows[2] + "\r" + rows[4] + "\r\n\r\n").encode())
    add("blank_then_error", ibm(rows + ["", "x"]))
    # whitespace (str.strip, unicode), keys: bank + account tuples
    add("strip_keys", ibm([" 5 ,\t1 , A ,1,B ,1, USD ,1,　USD ,Wire, 1 ",
                           "6,1,A,01,B,1,USD,1,USD,Wire,TRUE", "7,1 ,A,1,B,1,usd,1,usd,Wire,yes",
                           "8,1,A,1,b,1,USD,1,USD,Wire,No", "9,2,A,1,B,1,USD,1,USD,Wire,false",
                           "10,,A,,A,1,USD,1,,Wire,"]))
    add("bank_vs_none", b"Timestamp,From Bank,Account,Account,Is Laundering\n1,9,a,a,0\n2,9,a,9,1\n",
        dst_bank=None, amount=None, currency=None)
    # integers and datetimes
    add("int_forms", ibm(["+5,1,A,1,B,1,USD,1,USD,Wire,0", "0005,1,A,1,B,1,USD,1,USD,Wire,0",
                          "1_000,1,A,1,B,1,USD,1,USD,Wire,0", "-0,1,A,1,B,1,USD,1,USD,Wire,0",
                          " 9223372036854775807 ,1,A,1,B,1,USD,1,USD,Wire,0"]))
    add("negative_ts", ibm(["5,1,A,1,B,1,USD,1,USD,Wire,0", "-5,1,A,1,B,1,USD,1,USD,Wire,0"]))
    add("negative_ts_int_only", ibm(["-7,1,A,1,B,1,USD,1,USD,Wire,0"]), timestamp_format=None)
    add("no_format", ibm(["2022/09/01 00:20,1,A,1,B,1,USD,1,USD,Wire,0"]), timestamp_format=None)
    add("datetime_forms", ibm(["2022/9/1 0:5,1,A,1,B,1,USD,1,USD,Wire,0",
                               "2020/02/29 23:59,1,A,1,B,1,USD,1,USD,Wire,0",
                               "1970/01/01 00:00,1,A,1,B,1,USD,1,USD,Wire,0",
                               "2022/09/01   00:20,1,A,1,B,1,USD,1,USD,Wire,0",
                               "9999/12/31 23:59,1,A,1,B,1,USD,1,USD,Wire,0"]))
    add("datetime_feb30", ibm(["2022/02/30 00:00,1,A,1,B,1,USD,1,USD,Wire,0"]))
    add("datetime_pre_epoch", ibm(["1969/12/31 23:59,1,A,1,B,1,USD,1,USD,Wire,0"]))
    add("datetime_unconverted", ibm(["2022/09/01 00:201,1,A,1,B,1,USD,1,USD,Wire,0"]))
    add("datetime_year0", ibm(["0000/01/01 00:00,1,A,1,B,1,USD,1,USD,Wire,0"]))
    add("datetime_seconds", ibm(["2022-09-01T00:20:59,1,A,1,B,1,USD,1,USD,Wire,0",
                                 "2022-9-1t1:2:3,1,A,1,B,1,USD,1,USD,Wire,0"]),
        timestamp_format="%Y-%m-%dT%H:%M:%S", tick_seconds=7)
    add("datetime_leap_second", ibm(["2022-09-01T00:20:60,1,A,1,B,1,USD,1,USD,Wire,0"]),
        timestamp_format="%Y-%m-%dT%H:%M:%S")
    add("datetime_compact", ibm(["202209010020,1,A,1,B,1,USD,1,USD,Wire,0",
                                 "22091 0 5,1,A,1,B,1,USD,1,USD,Wire,0"]), timestamp_format="%Y%m%d%H%M")
    add("datetime_2digit_year", ibm(["68/1/2 3:04,1,A,1,B,1,USD,1,USD,Wire,0",
                                     "69/1/2 3:04,1,A,1,B,1,USD,1,USD,Wire,0"]), timestamp_format="%y/%m/%d %H:%M")
    add("datetime_day_space", ibm(["2022/09/ 1 00:20,1,A,1,B,1,USD,1,USD,Wire,0"]))
    # amounts (float(): correctly rounded)
    amounts = ["3697.34", "0.1", "5530.170593218375", "1e5", "1E-05", "-0", ".5", "5.", " 12 ", "+7.25",
               "inf", "-Infinity", "1234567890123456789", "0.000000000000000000001", "9007199254740993",
               "123456789012345678e-10", "2.2250738585072014e-08", "1.7976931348623157e1", "00042.4200",
               "4.35", "0.30000000000000004", "1e19", "17976931348623157e-16"]
    add("amounts", ibm([f"{i},1,A,1,B,1,USD,{a},USD,Wire,0" for i, a in enumerate(amounts)]))
    add("amount_nan", ibm(["1,1,A,1,B,1,USD,nan,USD,Wire,0", "2,1,A,1,B,1,USD,-NaN,USD,Wire,0"]))
    add("amount_bad", ibm(["1,1,A,1,B,1,USD,12.5,USD,Wire,0", "2,1,A,1,B,1,USD,12,5,USD,Wire,0"]))
    add("amount_bad2", ibm(["1,1,A,1,B,1,USD,1e,USD,Wire,0"]))
    add("amount_empty", ibm(["1,1,A,1,B,1,USD,,USD,Wire,0"]))
    add("label_bad", ibm(["1,1,A,1,B,1,USD,1,USD,Wire,0", "2,1,A,1,B,1,USD,1,USD,Wire,maybe"]))
    add("error_order", ibm(["x,1,A,1,B,1,USD,bad,USD,Wire,maybe"]))
    add("error_order2", ibm(["-1,1,A,1,B,1,USD,bad,USD,Wire,maybe"]))
    add("error_order3", ibm(["1,1,A,1,B,1,USD,bad,USD,Wire,maybe"]))
    add("dup_header", b"t;acc;acc;acc;amt\n1;a;b;c;2.5\n2;c;a;b;3\n",
        timestamp="t", src_bank=None, src_account="acc", dst_bank=None, dst_account="acc", amount="amt",
        currency=None, label=None, delimiter=";")
    add("tab_delim", b"Timestamp\tAccount\tAccount\n3\tx\ty\n4\ty\tx\n", src_bank=None, dst_bank=None,
        amount=None, currency=None, label=None, delimiter="\t")
    add("extra_columns", ibm(["1,1,A,1,B,1,USD,1,USD,Wire,0,extra,fields", "2,1,A,1,B,1,USD,1,USD,Wire,0"]))
    # reference synth.write_csv output (integer ticks, repr-float amounts)
    for seed, (n, e) in enumerate([(40, 300), (300, 3000), (1500, 20000)]):
        cfg = rsynth.SynthConfig(n, e, 50_000, seed=11 + seed,
                                 plants=(rsynth.PlantSpec("sg_count", 3, (3, 4), 300),
                                         rsynth.PlantSpec("cycle_3", 2, span=300)))
        records, _ = rsynth.generate(cfg)
        path = Path(f"/tmp/_ingest_synth_{seed}.csv")
        rsynth.write_csv(records, str(path))
        add(f"synth_{n}_{e}", path.read_bytes())
    # a random IBM-like log with datetimes, banks, currencies and labels
    rng = random.Random(7)
    cur = ["US Dollar", "Euro", "Yuan", "Bitcoin", "Rupee", "UK Pound"]
    rows = []
    for i in range(4000):
        b1, b2 = rng.randint(0, 40), rng.randint(0, 40)
        a1, a2 = f"{rng.randint(0, 800):08X}", f"{rng.randint(0, 800):08X}"
        ts = f"2022/09/{rng.randint(1, 18):02d} {rng.randint(0, 23):02d}:{rng.randint(0, 59):02d}"
        amt = f"{rng.uniform(0.01, 2e6):.2f}"
        c = rng.choice(cur)
        rows.append(f"{ts},{b1:03d},{a1},{b2:03d},{a2},{amt},{c},{amt},{c},ACH,{rng.random() < 0.01:d}")
    add("ibm_like_4000", ibm(rows))
    return out


def run_reference(data: bytes, mapping: dict):
    import io
    m = ColumnMapping(**mapping)
    try:
        records = parse_transactions(io.StringIO(data.decode("utf-8"), newline=""), m)
        g = build_graph(records)
    except Exception as exc:  # the error is the expected result
        return {"error": type(exc).__name__, "line": getattr(exc, "line", None), "message": str(exc)}, None
    arrays = {"src": g.edge_src, "dst": g.edge_dst, "time": g.edge_time,
              "amount_bits": g.edge_amount.view(np.uint64), "currency": g.edge_currency, "label": g.edge_label}
    return {"n_edges": int(g.edge_count), "node_count": int(g.node_count), "vocab": list(g.currency_vocab)}, arrays


def main():
    meta = []
    arrays = {}
    for k, (name, data, mapping) in enumerate(cases()):
        res, arr = run_reference(data, mapping)
        meta.append({"name": name, "mapping": mapping, **res})
        arrays[f"csv{k}"] = np.frombuffer(data, dtype=np.uint8)
        if arr is not None:
            for key, a in arr.items():
                arrays[f"{key}{k}"] = np.asarray(a)
        print(f"{k:3d} {name:24s} {res.get('error') or res['n_edges']} {res.get('message', '')[:70]}")
    # the reference's cache file (cache.save_graph, cache.py:40-52) of one case
    import io
    import tempfile
    from tempmine import cache as rcache
    k = [m["name"] for m in meta].index("ibm_like_4000")
    g = build_graph(parse_transactions(io.StringIO(bytes(arrays[f"csv{k}"]).decode(), newline="")))
    with tempfile.TemporaryDirectory() as d:
        rcache.save_graph(g, f"{d}/g.tmg")
        arrays["cache_bytes"] = np.frombuffer(Path(f"{d}/g.tmg").read_bytes(), dtype=np.uint8)
    arrays["cache_case"] = np.array(k)
    np.savez_compressed(OUT, meta=json.dumps(meta), **arrays)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
