import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1503_07387_b200 import _lib, mvb, workload as W
dev = torch.device("cuda", 0)
w = W.config2()
nset = 4
srcs = [torch.from_numpy(w.encoded).to(dev) for _ in range(nset)]
outs = [torch.empty(w.count, dtype=torch.int32, device=dev) for _ in range(nset)]
d = mvb.Decoder(dev, w.encoded.size)
def run(k): d.decode_delta(srcs[k % nset], w.count, w.prev, outs[k % nset])
for k in range(20): run(k)
torch.cuda.synchronize()
for mode in ("plain", "events", "plain", "events"):
    n = 50
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for k in range(n):
        if mode == "events": evs[k][0].record()
        run(k)
        if mode == "events": evs[k][1].record()
    e.record(); torch.cuda.synchronize()
    tot = s.elapsed_time(e) * 1e3 / n
    per = np.mean([a.elapsed_time(b) for a, b in evs]) * 1e3 if mode == "events" else 0
    print(f"{mode:7s} total/decode {tot:6.1f} us  per-event-pair {per:6.1f} us")
