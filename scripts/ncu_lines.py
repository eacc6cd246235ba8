"""Executed warp instructions and stall samples aggregated per CUDA source line."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
cur_file = None
func = None
agg = defaultdict(lambda: [0, 0, ""])
hdr = None
cur_line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        if func is not None and r[1] != func:
            break
        func = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    d = dict(zip(hdr[2:], r[2:]))
    if r[0]:
        cur_line = (cur_file, int(r[0]), r[1][:70])
    if not d.get("Address"):
        continue
    try:
        n = int(d.get("Instructions Executed") or 0)
        st = int(d.get("Warp Stall Sampling (All Samples)") or 0)
    except ValueError:
        continue
    a = agg[cur_line[:2]]
    a[0] += n
    a[1] += st
    a[2] = cur_line[2]
tot = sum(v[0] for v in agg.values()) or 1
stot = sum(v[1] for v in agg.values()) or 1
print("total", tot, "function", func)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * v[0] / tot:5.1f}% instr {100 * v[1] / stot:5.1f}% stall  {k[0]}:{k[1]:<4d} {v[2]}")
