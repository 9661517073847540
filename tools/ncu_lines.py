"""Stall samples per CUDA source line from an ncu report (run here, no GPU):
    python tools/ncu_lines.py REP.ncu-rep KERNEL_REGEX [top=30]
Uses the mixed cuda,sass source page (needs -lineinfo builds)."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
agg = defaultdict(lambda: [0, ""])
fname = "?"
cur = None
head = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        head = row
        si = head.index("Warp Stall Sampling (All Samples)")
        continue
    if head is None or len(row) <= si:
        continue
    if row[0]:
        cur = (fname, int(row[0]))
        agg[cur][1] = row[1].strip()[:90]
        try:
            agg[cur][0] += int(row[si])  # line rows carry the line's total
        except ValueError:
            pass
tot = sum(v[0] for v in agg.values()) or 1
print(f"total samples {tot}")
for (f, ln), (n, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{n:8d} {100 * n / tot:5.1f}%  {f}:{ln:<5d} {src}")
