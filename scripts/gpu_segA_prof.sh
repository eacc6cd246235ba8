#!/bin/bash
mkdir -p gpurun_out
python /tmp/seg_run.py c2 >/dev/null 2>&1 || cat > /tmp/seg_run.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1503_07387_b200 import _lib, mvb, workload as W
_lib.set_kernel_choice(int(sys.argv[2]) if len(sys.argv) > 2 else 4)
w = {"c2": W.config2, "c1": W.config1, "all1": lambda: W.config5("all1")}[sys.argv[1]]()
dev = torch.device("cuda", 0)
src = torch.from_numpy(w.encoded).to(dev); out = torch.empty(w.count, dtype=torch.int32, device=dev)
d = mvb.Decoder(dev, w.encoded.size)
for it in range(6):
    if w.delta: d.decode_delta(src, w.count, w.prev, out)
    else: d.decode(src, w.count, out)
torch.cuda.synchronize()
print("ok", d.result())
PY
python /tmp/seg_run.py c2 > gpurun_out/seg_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:seg_totals -s 3 -c 1 -o gpurun_out/prof_segA python /tmp/seg_run.py c2 > gpurun_out/ncu_segA.log 2>&1; echo ncu rc=$?
