"""Histogram of SASS instructions of one kernel by execution count (per-launch):
how many static instructions run ~N times, and the executed total per bucket.
usage: ncu_sass_counts.py REP KERNEL_REGEX"""
import csv, io, subprocess, sys, collections
rep, kern = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kern, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = next(r for r in rows if "Source" in r)
ix = {k: i for i, k in enumerate(hdr)}
body = [r for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
cnt = []
for r in body:
    try:
        c = int(r[ix["Instructions Executed"]] or 0)
    except ValueError:
        continue
    cnt.append((c, r[ix["Source"]].strip(), r[ix["Address"]] if "Address" in ix else ""))
tot = sum(c for c, _, _ in cnt)
b = collections.defaultdict(lambda: [0, 0])
for c, s, a in cnt:
    if c == 0:
        continue
    k = 1 << (c.bit_length() - 1)
    b[k][0] += 1
    b[k][1] += c
print("total executed", tot)
for k in sorted(b):
    print(f"count in [{k:>12}, {2*k:>12}): {b[k][0]:6d} static instrs, {b[k][1]:>14} executed ({100*b[k][1]/tot:5.1f}%)")
if len(sys.argv) > 3:
    lo, hi = int(sys.argv[3]), int(sys.argv[4])
    ops = collections.Counter()
    for c, s, a in cnt:
        if lo <= c < hi:
            t = s.split()
            op = t[1] if t[0].startswith("@") else t[0]
            ops[op.split(".")[0]] += 1
    print(ops.most_common(30))
