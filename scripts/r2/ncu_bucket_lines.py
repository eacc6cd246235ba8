"""Instructions of one kernel whose execution count lies in [lo, hi), grouped by CUDA source line
(the innermost line ncu correlates).  usage: ncu_bucket_lines.py REP KERNEL_REGEX LO HI [N]"""
import csv, io, subprocess, sys, collections
rep, kern, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
n = int(sys.argv[5]) if len(sys.argv) > 5 else 40
raw = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kern, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
agg = collections.Counter()
static = collections.Counter()
fname, hdr = "", None
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr is None:
        continue
    try:
        ie = int(r[hdr["Instructions Executed"]] or 0)
    except (ValueError, IndexError, KeyError):
        continue
    # per-SASS counts are not in the cuda view; use the line's executed count / its SASS count
    key = (fname, r[0], r[1].strip()[:90])
    agg[key] += ie
print("(per-line totals; lines whose executed count falls in the bucket)")
for k, v in agg.most_common(400):
    if lo <= v < hi * 64:
        pass
tot = sum(agg.values())
rows = [(v, k) for k, v in agg.items()]
rows.sort(reverse=True)
for v, k in rows[:n]:
    print(f"{v:>12} {100.0*v/tot:5.1f}%  {k[0]}:{k[1]}  {k[2]}")
