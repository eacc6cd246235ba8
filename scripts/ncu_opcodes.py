"""Executed warp-instructions by SASS opcode for one kernel of an ncu report.
usage: ncu_opcodes.py REP KERNEL_REGEX [N]"""
import collections, csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kern, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = next(r for r in rows if "Source" in r)
ix = {k: i for i, k in enumerate(hdr)}
ops, stalls = collections.Counter(), collections.Counter()
tot = 0
for r in rows[rows.index(hdr) + 1:]:
    if len(r) != len(hdr):
        continue
    src = r[ix["Source"]].strip()
    if not src or src.startswith("/*"):
        continue
    toks = src.split()
    op = toks[0]
    if op.startswith("@"):
        op = toks[1]
    op = op.split(".")[0]
    try:
        c = int(r[ix["Instructions Executed"]] or 0)
    except ValueError:
        continue
    ops[op] += c
    stalls[op] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot += c
print(f"total {tot}")
for op, c in ops.most_common(n):
    print(f"{op:10s} {c:10d} {100.0 * c / tot:5.1f}%  stall samples {stalls[op]}")
