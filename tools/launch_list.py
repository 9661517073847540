"""Aggregate an ncu launch list of a bench command, e.g.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file L.csv python bench.py --steps 1 --warmup 0 ...

per kernel of the LAST mining call (from the last k_lo_table launch):
launches, total ms, share, DRAM bytes.  With --config NAME the step's DRAM
bytes (read + write, all kernels of that call) go to
profiles/ncu_traffic.json[NAME]["step_dram_bytes"] (bench.py: roofline.traffic).

    python tools/launch_list.py L.csv [--config hi-large] [--md out.md]
"""
import argparse
import collections
import csv
import json
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SC = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3,
      "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def load(path):
    """[(launch id, kernel, {metric: value (ms / bytes)})] in launch order."""
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ii, ki = h.index("ID"), h.index("Kernel Name")
    mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        key = r[ii]
        if key not in out:
            out[key] = (r[ki].split("(")[0].split("::")[-1][:40], {})
        try:
            out[key][1][r[mi]] = float(r[vi].replace(",", "")) * SC.get(r[ui], 1)
        except ValueError:
            pass
    return [(k, n, m) for k, (n, m) in out.items()]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--last", default="k_lo_table")
    ap.add_argument("--config")
    ap.add_argument("--md")
    a = ap.parse_args()
    order = load(a.csv)
    starts = [i for i, (_, k, _) in enumerate(order) if k == a.last]
    sub = order[starts[-1] if starts else 0:]
    agg = collections.OrderedDict()
    for _, k, m in sub:
        x = agg.setdefault(k, [0, 0.0, 0.0])
        x[0] += 1
        x[1] += m.get("gpu__time_duration.sum", 0.0)
        x[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(x[1] for x in agg.values())
    dram = sum(x[2] for x in agg.values())
    lines = [f"last mining call (from the last {a.last}): {tot:.3f} ms, DRAM {dram / 1e9:.2f} GB",
             "", "| kernel | launches | ms | share | DRAM GB |", "|---|---|---|---|---|"]
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {k} | {n} | {t:.3f} | {100 * t / tot:.1f}% | {b / 1e9:.2f} |")
    print("\n".join(lines))
    if a.md:
        Path(a.md).write_text("\n".join(lines) + "\n")
    if a.config and dram > 0:
        tj = ROOT / "profiles" / "ncu_traffic.json"
        cur = json.loads(tj.read_text()) if tj.exists() else {}
        ent = cur.setdefault(a.config, {})
        ent["step_dram_bytes"] = dram
        ent["step_ms_ncu"] = tot
        ent["source"] = f"{Path(a.csv).name}: dram__bytes_read.sum + dram__bytes_write.sum over every kernel of one mining call"
        tj.write_text(json.dumps(cur, indent=1) + "\n")


if __name__ == "__main__":
    main()
