#!/bin/bash
# kernel time of strict kernel variants (default 0 and 5) on the SURVEY configs (L2 flushed before each launch)
CHOICES=${CHOICES:-"0 5"} python - <<'PY'
import os, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1503_07387_b200 import _lib, mvb, workload as W
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
choices = [int(c) for c in os.environ["CHOICES"].split()]
cfgs = {"c2": W.config2(), "c1": W.config1(), "all1": W.config5("all1"), "all5": W.config5("all5"),
        "p50": W.config5("p50"), "p50d": W.config5("p50", delta=True)}
for name, w in cfgs.items():
    src = torch.from_numpy(w.encoded).to(dev); out = torch.empty(w.count, dtype=torch.int32, device=dev)
    d = mvb.Decoder(dev, w.encoded.size); exp = torch.from_numpy(w.expected().view(np.int32)).to(dev)
    row = []
    for ch in choices:
        _lib.set_kernel_choice(ch)
        ts = []
        for it in range(15):
            flush.fill_(it); s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            out.fill_(-1)
            s.record()
            if w.delta: d.decode_delta(src, w.count, w.prev, out)
            else: d.decode(src, w.count, out)
            e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
        ok = torch.equal(out, exp)
        row.append(f"k{ch}={np.median(ts[3:]):7.1f}{'' if ok else '!BAD'}")
    print(f"{name:5s} n={w.count} bytes={w.encoded.size}", " ".join(row), flush=True)
_lib.set_kernel_choice(0)
PY
