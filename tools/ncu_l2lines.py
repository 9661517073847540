"""L2 sectors (global + local) per CUDA source line from an ncu report:
    python tools/ncu_l2lines.py REP.ncu-rep KERNEL_REGEX [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
agg = defaultdict(lambda: [0.0, 0.0, ""])
fname, head = "?", None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        head = row
        continue
    if head is None or len(row) != len(head):
        continue
    try:
        g = float(row[head.index("L2 Theoretical Sectors Global")] or 0)
        loc = float(row[head.index("L2 Theoretical Sectors Local")] or 0)
    except ValueError:
        continue
    k = f"{fname}:{row[0]}"
    agg[k][0] += g
    agg[k][1] += loc
    agg[k][2] = row[1][:90]
tot = sum(v[0] + v[1] for v in agg.values()) or 1
print(f"total L2 sectors {tot:.3e}")
for k, (g, l, src) in sorted(agg.items(), key=lambda kv: -(kv[1][0] + kv[1][1]))[:top]:
    print(f"{g + l:12.3e} {100 * (g + l) / tot:5.1f}%  global {g:10.3e} local {l:10.3e}  {k:22s} {src}")
