"""SASS of one kernel in address order with executed-instruction counts and the
CUDA source line each instruction maps to (ncu --print-source cuda,sass);
only instructions executed at least MIN times.  usage: ncu_sass_flow.py REP KERNEL_REGEX [MIN]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
mn = int(sys.argv[3]) if len(sys.argv) > 3 else 1
raw = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kern, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
items = []
fname, line = "", ""
ie_col = None
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        ie_col = r.index("Instructions Executed")
        continue
    if r[0] == "Function Name" or ie_col is None:
        continue
    if r[0]:
        line = f"{fname}:{r[0]}"
        continue
    try:
        items.append((int(r[2], 16), int(r[ie_col] or 0), r[3].strip(), line))
    except (ValueError, IndexError):
        pass
seen = {}
for it in items:  # an inlined instruction is listed under every source line it maps to: keep the innermost
    seen[it[0]] = it
items = sorted(seen.values())
tot = sum(i[1] for i in items)
print("total", tot)
for a, ie, s, l in items:
    if ie >= mn:
        print(f"{a & 0xFFFFF:05x} {ie:9d}  {s[:70]:70s} {l}")
