#!/bin/bash
# one ncu --set full capture of the segment decode kernel (kernel B) for CFG (c2/c1/all1) and CHOICE,
# after the same command has run clean without ncu
CFG=${CFG:-c2}; CHOICE=${CHOICE:-5}; TAG=${TAG:-ll}
mkdir -p gpurun_out
cat > /tmp/seg_run.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1503_07387_b200 import _lib, mvb, workload as W
_lib.set_kernel_choice(int(sys.argv[2]))
w = {"c2": W.config2, "c1": W.config1, "all1": lambda: W.config5("all1"), "all5": lambda: W.config5("all5"),
     "p50": lambda: W.config5("p50")}[sys.argv[1]]()
dev = torch.device("cuda", 0)
src = torch.from_numpy(w.encoded).to(dev); out = torch.empty(w.count, dtype=torch.int32, device=dev)
d = mvb.Decoder(dev, w.encoded.size)
for it in range(6):
    if w.delta: d.decode_delta(src, w.count, w.prev, out)
    else: d.decode(src, w.count, out)
torch.cuda.synchronize()
assert np.array_equal(out.cpu().numpy().view(np.uint32), w.expected()), "mismatch"
print("ok", d.result())
PY
python /tmp/seg_run.py $CFG $CHOICE > gpurun_out/ll_run.log 2>&1 && \
ncu --set full --clock-control none ${NCU_EXTRA:-} --import-source on -k regex:"seg_decode|seg_totals|seg_fused" -s 4 -c 2 -o gpurun_out/prof_$TAG python /tmp/seg_run.py $CFG $CHOICE > gpurun_out/ncu_$TAG.log 2>&1; echo ncu rc=$?
cat gpurun_out/ll_run.log
