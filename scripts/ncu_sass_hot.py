"""Top SASS instructions of an ncu report by warp-stall samples, with a few
neighbouring instructions for context, plus shared-memory wavefront excess
per instruction.  usage: ncu_sass_hot.py REP [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ix = {k: i for i, k in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
inst = sum(int(r[ix["Instructions Executed"]] or 0) for r in body)
wf = sum(int(r[ix["L1 Wavefronts Shared"]] or 0) for r in body) if "L1 Wavefronts Shared" in ix else 0
wfi = sum(int(r[ix["L1 Wavefronts Shared Ideal"]] or 0) for r in body) if "L1 Wavefronts Shared Ideal" in ix else 0
print(f"samples {tot}  instructions {inst}  smem wavefronts {wf} (ideal {wfi})")
order = sorted(range(len(body)), key=lambda i: -int(body[i][ix["Warp Stall Sampling (All Samples)"]] or 0))
for i in order[:n]:
    r = body[i]
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    print(f"{100.0 * s / tot:5.1f}%  [{i:5d}] exec {r[ix['Instructions Executed']]:>8s}  {r[ix['Source']].strip()[:70]}")
print("-- smem wavefronts by instruction (top)")
order = sorted(range(len(body)), key=lambda i: -int(body[i][ix["L1 Wavefronts Shared"]] or 0))
for i in order[:n]:
    r = body[i]
    print(f"[{i:5d}] wf {r[ix['L1 Wavefronts Shared']]:>8s} ideal {r[ix['L1 Wavefronts Shared Ideal']]:>8s}  exec {r[ix['Instructions Executed']]:>8s}  {r[ix['Source']].strip()[:60]}")
