"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launches / total ms, and the kernels of the last mining call.

    python tools/launch_list.py gpurun_out/launches.csv [--last k_lo_table]
"""
import collections
import csv
import sys

SC = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        out.append((r[ki].split("(")[0].split("::")[-1][:40], float(r[vi].replace(",", "")) * SC[r[ui]]))
    return out


def main():
    path = sys.argv[1]
    first = sys.argv[sys.argv.index("--last") + 1] if "--last" in sys.argv else "k_lo_table"
    order = load(path)
    starts = [i for i, (k, _) in enumerate(order) if k == first]
    idx = starts[-1] if starts else 0
    sub = order[idx:]
    agg = collections.OrderedDict()
    for k, t in sub:
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += t
    tot = sum(a[1] for a in agg.values())
    print(f"last mining call (from the last {first}): {tot:.3f} ms")
    print("| kernel | launches | ms | share |\n|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {n} | {t:.3f} | {100 * t / tot:.1f}% |")


if __name__ == "__main__":
    main()
