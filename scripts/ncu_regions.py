"""Executed warp instructions per CUDA source line range (from sass,cuda view):
prints each source line with its executed instruction total, in source order,
for lines above a threshold."""
import csv
import io
import subprocess
import sys
from collections import OrderedDict

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.003
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = None
cur = None
cf = None
func = None
agg = OrderedDict()
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
        cur = (cf, int(r[0]))
        if cur not in agg:
            agg[cur] = [0, r[1][:80]]
        continue
    d = dict(zip(hdr[2:], r[2:]))
    if not d.get("Address") or cur is None:
        continue
    try:
        agg[cur][0] += int(d.get("Instructions Executed") or 0)
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values()) or 1
print("total", tot)
for (f, ln), (n, src) in sorted(agg.items(), key=lambda kv: (kv[0][0], kv[0][1])):
    if n > thr * tot:
        print(f"{100 * n / tot:5.1f}%  {f}:{ln:<4d} {src}")
