"""Per CUDA source line of one kernel: warp-stall samples by reason (deduped by
SASS address, attributed to the innermost source line).
usage: ncu_stall_lines.py REP KERNEL_REGEX [N]"""
import csv, io, subprocess, sys, collections

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kern, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
reasons = ["stall_barrier", "stall_branch_resolving", "stall_dispatch", "stall_lg", "stall_long_sb", "stall_math",
           "stall_mio", "stall_no_inst", "stall_not_selected", "stall_selected", "stall_short_sb", "stall_wait"]
fname, line, hdr = "", "", None
seen = {}
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
        line = f"{fname}:{r[0]}"
        continue
    try:
        seen[r[2]] = (line, {k: int(r[hdr[k]] or 0) for k in reasons})
    except (ValueError, IndexError, KeyError):
        pass
agg = collections.defaultdict(collections.Counter)
for line, d in seen.values():
    agg[line].update(d)
tot = sum(sum(c.values()) for c in agg.values())
print("total samples", tot)
for line, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:n]:
    s = sum(c.values())
    top = ", ".join(f"{k[6:]} {v}" for k, v in c.most_common(3) if v)
    print(f"{100.0 * s / tot:5.1f}%  {line:28s} {top}")
