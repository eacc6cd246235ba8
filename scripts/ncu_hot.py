"""Hot SASS blocks (runs of equal execution count) of the first kernel in an ncu report."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.005
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = None
data = []
seen = set()
for r in rows:
    if r and r[0] == "Address":
        if hdr is not None:
            break
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Address"] in seen:
            continue
        seen.add(d["Address"])
        data.append(d)
blocks = []
cur = None
for i, d in enumerate(data):
    n = int(d["Instructions Executed"] or 0)
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    if cur and cur[0] == n:
        cur[1] += 1
        cur[3] = d["Source"]
        cur[5] += s
    else:
        if cur:
            blocks.append(cur)
        cur = [n, 1, d["Source"], d["Source"], i, s]
blocks.append(cur)
tot = sum(b[0] * b[1] for b in blocks)
stot = sum(b[5] for b in blocks) or 1
print("total warp instructions", tot)
for b in blocks:
    if b[0] * b[1] > thr * tot or b[5] > 0.03 * stot:
        print(f"#{b[4]:5d} exec {b[0]:8d} x{b[1]:4d} = {100 * b[0] * b[1] / tot:5.1f}%  stall {100 * b[5] / stot:5.1f}%  "
              f"{b[2][:38]:38s} .. {b[3][:38]}")
