"""Ingestion throughput (GPU box): an IBM-layout CSV (datetime timestamps,
bank + account keys, 2-decimal and repr-float amounts, currencies, labels)
parsed by the GPU (ingest.read_transactions: bytes in host memory -> host
edge arrays; ingest.ingest_csv: -> device graph) and, on a bounded sample,
by the CPU restatement of the reference (oracle/ingest_oracle.py, the
reference's own algorithm: csv.reader + int/strptime/float + dicts).

    python tools/bench_ingest.py [n_rows=2000000]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402


def make_csv(n: int, seed: int = 2604) -> bytes:
    rng = np.random.default_rng(seed)
    n_acc = max(16, n // 10)
    acc_src = (rng.pareto(1.0, n) * 7).astype(np.int64) % n_acc
    acc_dst = rng.integers(0, n_acc, n)
    bank = rng.integers(0, 3000, (2, n))
    t = np.sort(rng.integers(0, 10 * 86400, n)) + 1661990400  # 2022/09/01
    day = (t - 1661990400) // 86400 + 1
    hh = (t % 86400) // 3600
    mm = (t % 3600) // 60
    amt = rng.uniform(0.01, 2e6, n)
    cur = np.array(["US Dollar", "Euro", "Yuan", "Bitcoin", "Rupee", "UK Pound", "Yen"])[rng.integers(0, 7, n)]
    lab = (rng.random(n) < 0.001).astype(int)
    head = ("Timestamp,From Bank,Account,To Bank,Account,Amount Received,Receiving Currency,Amount Paid,"
            "Payment Currency,Payment Format,Is Laundering")
    rows = [head]
    for i in range(n):
        a = f"{amt[i]:.2f}"
        rows.append(f"2022/09/{day[i]:02d} {hh[i]:02d}:{mm[i]:02d},{bank[0, i]:03d},{acc_src[i]:09X},"
                    f"{bank[1, i]:03d},{acc_dst[i]:09X},{a},{cur[i]},{a},{cur[i]},ACH,{lab[i]}")
    return ("\n".join(rows) + "\n").encode()


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
    t0 = time.perf_counter()
    data = make_csv(n)
    print(f"[bench_ingest] generated {n} rows, {len(data) / 1e6:.1f} MB in {time.perf_counter() - t0:.1f}s",
          file=sys.stderr)
    from paper_2604_12241_b200 import ingest
    best = {}
    for rep in range(4):
        t = time.perf_counter()
        tab = ingest.read_transactions(data)
        r = time.perf_counter() - t
        t = time.perf_counter()
        g = ingest.ingest_csv(data)
        c = time.perf_counter() - t
        g.free()
        if rep:
            best["read_s"] = min(best.get("read_s", 1e9), r)
            best["ingest_graph_s"] = min(best.get("ingest_graph_s", 1e9), c)
    # CPU: the reference algorithm on a bounded sample
    from oracle import ingest_oracle
    m = min(n, 200_000)
    cut = data.index(b"\n", int(len(data) * m / n)) + 1
    t = time.perf_counter()
    want = ingest_oracle.parse(data[:cut])
    cpu = time.perf_counter() - t
    sub = ingest.read_transactions(data[:cut])
    same = (np.array_equal(sub.edge_src, want["src"]) and np.array_equal(sub.edge_time, want["time"])
            and np.array_equal(sub.edge_amount.view(np.uint64), want["amount"].view(np.uint64)))
    rows_cpu = len(want["src"])
    print(json.dumps({
        "rows": n, "bytes": len(data), "nodes": tab.node_count,
        "gpu_read_transactions_s": round(best["read_s"], 4),
        "gpu_rows_per_s": n / best["read_s"], "gpu_GB_per_s": len(data) / best["read_s"] / 1e9,
        "gpu_ingest_csv_to_graph_s": round(best["ingest_graph_s"], 4),
        "cpu_reference_algorithm_rows_per_s": rows_cpu / cpu, "cpu_sample_rows": rows_cpu, "cpu_threads": 1,
        "sample_parity": bool(same),
        "note": "GPU times include H2D of the CSV bytes and D2H of the edge arrays (host in, host out)"}))


if __name__ == "__main__":
    main()
