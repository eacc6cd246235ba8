"""Time the default device decode of a config for several fused (segment bytes, lag %) settings:
python scripts/r2/sweep_chunk.py c4 4096:100 8192:50 ...
mvbx_set_fused_chunk): python scripts/r2/sweep_chunk.py c4 4194304 16777216 ..."""
import ctypes, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1503_07387_b200 import _lib, mvb
import bench
cfg = sys.argv[1]
w = bench.make_workload(cfg)
dev = torch.device("cuda", 0)
R = 3
srcs = [torch.from_numpy(w.encoded).to(dev) for _ in range(R)]
outs = [torch.empty(w.count, dtype=torch.int32, device=dev) for _ in range(R)]
d = mvb.Decoder(dev, capacity_bytes=int(w.encoded.size))
L = _lib.lib()
has_set = hasattr(L, "mvbx_set_fused")
if has_set:
    L.mvbx_set_fused.argtypes = [ctypes.c_size_t, ctypes.c_longlong]
exp = torch.from_numpy(w.expected().view(np.int32)).to(dev)
for arg in sys.argv[2:]:
    try:
        seg, lag = (int(x) for x in arg.split(":"))
    except ValueError:  # a label (library variant runs)
        seg, lag = arg, 0
    if has_set and isinstance(seg, int):
        L.mvbx_set_fused(seg, lag)
    def step(i):
        k = i % R
        if w.delta: d.decode_delta(srcs[k], w.count, w.prev, outs[k])
        else: d.decode(srcs[k], w.count, outs[k])
    step(0); torch.cuda.synchronize()
    ok = torch.equal(outs[0], exp)
    for i in range(5): step(i)
    torch.cuda.synchronize()
    n = 20 if w.count > 1 << 26 else 200
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n): step(i)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    alg = w.encoded.size + 4 * w.count
    print(f"{cfg} seg={seg} lag={lag}% ok={ok} {ms*1e3:.1f} us  {alg/ms/1e6:.0f} GB/s frac={alg/ms/1e6/6551:.3f}", flush=True)
