"""Stall samples per CUDA source line with the dominant reasons."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = None
cur = None
agg = defaultdict(lambda: defaultdict(int))
func = None
cf = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cf = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        if func and r[1] != func:
            break
        func = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if not hdr:
        continue
    if r[0]:
        cur = (cf, int(r[0]), r[1][:60])
    d = dict(zip(hdr[2:], r[2:]))
    if not d.get("Address"):
        continue
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                agg[cur][k] += int(v or 0)
            except ValueError:
                pass
tot = sum(sum(v.values()) for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:n]:
    s = sum(v.values())
    top = sorted(v.items(), key=lambda x: -x[1])[:3]
    print(f"{100 * s / tot:5.1f}% {k[0]}:{k[1]} {k[2][:55]:55s} " + " ".join(f"{a[6:]}={100 * b / s:.0f}%" for a, b in top))
