"""Summarize ncu captures into profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep --config hi-small --tag r01 \
        [--launches gpurun_out/launches.csv]

Writes profiles/ncu_<tag>_<config>.md (per-kernel table + top stall lines)
and merges {config: {kernel: {...}}} into profiles/ncu_traffic.json, which
bench.py reads for roofline.traffic (dram read + write bytes per launch).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
METRICS = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "regs",
    "smsp__inst_executed.sum": "warp_inst",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
              "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
              "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def raw(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[head.index("Kernel Name")].split("(")[0].split("::")[-1]}
        for m, key in METRICS.items():
            if m not in head:
                continue
            i = head.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if key in ("dram_read", "dram_write"):
                v *= UNIT_SCALE.get(u, 1)
            if key == "time":
                v *= UNIT_SCALE.get(u, 1)  # -> ms
            d[key] = v
        stalls = {}
        for i, name in enumerate(head):
            if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
                try:
                    stalls[name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(r[i])
                except ValueError:
                    pass
        d["top_stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:4])
        res.append(d)
    return res


def launches(path: str):
    text = Path(path).read_text()
    lines = [ln for ln in text.splitlines() if not ln.startswith("==")]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        k = r[ki].split("(")[0].split("::")[-1]
        agg[k][0] += 1
        agg[k][1] += float(r[vi].replace(",", "")) / 1e6  # ns -> ms
    return dict(agg)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--config", default="hi-small")
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--launches")
    a = ap.parse_args()
    ks = raw(a.rep)
    md = [f"# ncu summary — {a.tag}, workload {a.config}", "",
          f"source: `{a.rep}` (`ncu --set full --clock-control none`; cold-cache, serialised replay)", "",
          "| kernel | ms | DRAM read MB | DRAM write MB | L2 hit % | warps active % | regs | top stalls (per issue) |",
          "|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for d in ks:
        st = ", ".join(f"{k} {v:.1f}" for k, v in d["top_stalls"].items())
        md.append(f"| {d['kernel']} | {d.get('time', 0):.3f} | {d.get('dram_read', 0) / 1e6:.1f} | "
                  f"{d.get('dram_write', 0) / 1e6:.1f} | {d.get('l2_hit_pct', 0):.1f} | "
                  f"{d.get('warps_active_pct', 0):.1f} | {int(d.get('regs', 0))} | {st} |")
        traffic[d["kernel"]] = {"dram_bytes": d.get("dram_read", 0) + d.get("dram_write", 0),
                                "ms": d.get("time"), "l2_hit_pct": d.get("l2_hit_pct")}
    if a.launches:
        md += ["", "## launch list (gpu__time_duration.sum, all launches of the command)", "",
               "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        agg = launches(a.launches)
        tot = sum(v[1] for v in agg.values())
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            md.append(f"| {k} | {n} | {t:.3f} | {100 * t / tot:.1f}% |")
    out = ROOT / "profiles" / f"ncu_{a.tag}_{a.config}.md"
    out.write_text("\n".join(md) + "\n")
    tj = ROOT / "profiles" / "ncu_traffic.json"
    cur = json.loads(tj.read_text()) if tj.exists() else {}
    cur.setdefault(a.config, {})["kernels"] = traffic  # per-kernel; launch_list.py adds step_dram_bytes
    tj.write_text(json.dumps(cur, indent=1) + "\n")
    print(out.read_text())


if __name__ == "__main__":
    main()
