"""Instructions executed and stall samples per CUDA source line of one kernel
of an ncu report (ncu -i REP -k regex:KERNEL --page source --print-source cuda,sass).
usage: ncu_lines.py REP KERNEL_REGEX [N]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kern, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
lines = {}
fname = ""
hdr = None
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r) if k not in ("Source",)}
        hdr["Instructions Executed"] = r.index("Instructions Executed")
        hdr["Warp Stall Sampling (All Samples)"] = r.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    try:
        ie = int(r[hdr["Instructions Executed"]] or 0)
        st = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, IndexError):
        continue
    key = (fname, int(r[0]), r[1].strip()[:80])
    a = lines.setdefault(key, [0, 0])
    a[0] += ie
    a[1] += st
# note: inlined instructions count once per source line they map to (totals exceed the kernel's)
ti = sum(v[0] for v in lines.values())
ts = sum(v[1] for v in lines.values())
print(f"total instructions {ti}  stall samples {ts}")
for k, v in sorted(lines.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{100.0 * v[0] / ti:5.1f}% inst {100.0 * v[1] / max(ts, 1):5.1f}% stall  {k[0]}:{k[1]}  {k[2]}")
