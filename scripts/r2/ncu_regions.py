"""Executed warp-instructions of one kernel grouped into named source regions (file:line ranges).
usage: ncu_regions.py REP KERNEL_REGEX  (regions below are those of decode_fused.cuh / decode_seg.cuh)"""
import csv, io, subprocess, sys, collections
rep, kern = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kern, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
fname, line, hdr = "", None, None
per = collections.Counter()
seen = set()
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0]:
        line = (fname, int(r[0]))
        continue
    try:
        addr = r[2]
        if addr in seen:
            continue
        seen.add(addr)
        per[line] += int(r[hdr["Instructions Executed"]] or 0)
    except (ValueError, IndexError, KeyError):
        pass
tot = sum(per.values())
print("total warp instructions", tot)
import re
regions = []
for spec in sys.argv[3:]:
    name, f, lo, hi = spec.split(":")
    regions.append((name, f, int(lo), int(hi)))
agg = collections.Counter()
for (f, l), v in per.items():
    for name, rf, lo, hi in regions:
        if f == rf and lo <= l <= hi:
            agg[name] += v
            break
    else:
        agg[f"other:{f}"] += v
for k, v in agg.most_common():
    print(f"{v:>12} {100.0*v/tot:5.1f}%  {k}")
