#!/bin/bash
# decode time of strict kernel variants (CHOICES, default "0 5") on the SURVEY configs: mean over 24
# back-to-back decodes cycling through buffer sets whose total exceeds L2 (as bench.py), after a
# correctness check of every variant
CHOICES=${CHOICES:-"0 5"} CFGS=${CFGS:-"c2 c1 all1 all5 p50 p50d"} python - <<'PY'
import os, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1503_07387_b200 import _lib, mvb, workload as W
dev = torch.device("cuda", 0)
choices = [int(c) for c in os.environ["CHOICES"].split()]
mk = {"c2": W.config2, "c1": W.config1, "all1": lambda: W.config5("all1"), "all5": lambda: W.config5("all5"),
      "p50": lambda: W.config5("p50"), "p50d": lambda: W.config5("p50", delta=True),
      "c4s": lambda: W.config4(n=1 << 27), "c4": W.config4}
for name in os.environ["CFGS"].split():
    w = mk[name]()
    per = w.encoded.size + 4 * w.count
    nset = max(2, -(-(300 << 20) // per))
    srcs = [torch.from_numpy(w.encoded).to(dev) for _ in range(nset)]
    outs = [torch.empty(w.count, dtype=torch.int32, device=dev) for _ in range(nset)]
    d = mvb.Decoder(dev, w.encoded.size)
    exp = torch.from_numpy(w.expected().view(np.int32)).to(dev)
    row = []
    for ch in choices:
        _lib.set_kernel_choice(ch)
        def run(k):
            if w.delta: d.decode_delta(srcs[k % nset], w.count, w.prev, outs[k % nset])
            else: d.decode(srcs[k % nset], w.count, outs[k % nset])
        outs[0].fill_(-1); run(0); torch.cuda.synchronize()
        ok = torch.equal(outs[0], exp)
        for k in range(4): run(k)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record()
        for k in range(24): run(k)
        e.record(); torch.cuda.synchronize()
        row.append(f"k{ch}={s.elapsed_time(e) * 1e3 / 24:7.1f}{'' if ok else '!BAD'}")
    print(f"{name:5s} n={w.count} bytes={w.encoded.size} sets={nset}", " ".join(row), flush=True)
    del srcs, outs
_lib.set_kernel_choice(0)
PY
