"""SASS of one kernel with per-instruction execution counts (warp-level).
usage: ncu_sass_dump.py REP KERNEL_REGEX > out.txt"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kern, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = next(r for r in rows if "Source" in r)
ix = {k: i for i, k in enumerate(hdr)}
seen = set()
for r in rows[rows.index(hdr) + 1:]:
    if len(r) != len(hdr):
        continue
    try:
        c = int(r[ix["Instructions Executed"]] or 0)
    except ValueError:
        continue
    addr = r[ix["Address"]] if "Address" in ix else ""
    if addr in seen:
        continue
    seen.add(addr)
    st = r[ix["Warp Stall Sampling (All Samples)"]]
    print(f"{addr:>8s} {c:9d} {st:>5s}  {r[ix['Source']].strip()}")
