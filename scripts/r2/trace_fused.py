"""Per-warp timeline of the fused decoder (a -DMVB_F_TRACE=1 build selected by MVB_CUDA_LIB):
python scripts/r2/trace_fused.py c2  -- when, relative to the first warp's start, the events happen
(1 start, 2 previous grid complete, 3 ticket, 4 unit landed, 5 published, 6 prefix known, 7 decoded, 8 done)."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1503_07387_b200 import _lib, mvb
import bench
cfg = sys.argv[1]
w = bench.make_workload(cfg)
dev = torch.device("cuda", 0)
src = torch.from_numpy(w.encoded).to(dev)
src2 = torch.from_numpy(w.encoded).to(dev)
out = torch.empty(w.count, dtype=torch.int32, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
d = mvb.Decoder(dev, capacity_bytes=int(w.encoded.size))
L = _lib.lib()
rows = torch.zeros(592 * 4 * 64, dtype=torch.int64, device=dev)
def step(s):
    if w.delta: d.decode_delta(s, w.count, w.prev, out)
    else: d.decode(s, w.count, out)
for _ in range(3): step(src)
torch.cuda.synchronize()
L.mvbx_set_fused_trace.argtypes = [ctypes.c_void_p]
for back_to_back in (0, 1):
    rows.zero_(); flush.fill_(1); torch.cuda.synchronize()
    assert L.mvbx_set_fused_trace(rows.data_ptr()) == 0
    if back_to_back:
        L.mvbx_set_fused_trace(None); step(src2); L.mvbx_set_fused_trace(rows.data_ptr())  # (a decode right before the traced one)
    step(src)
    torch.cuda.synchronize()
    r = rows.cpu().numpy().view(np.uint64).reshape(-1, 64)
    n = r[:, 0].astype(int)
    ev = [[(int(x) >> 4, int(x) & 15) for x in r[i, 1:1 + n[i]]] for i in range(r.shape[0]) if n[i]]
    t0 = min(e[0][0] for e in ev)
    print(f"== {cfg} back_to_back={back_to_back}: {len(ev)} warps")
    for code, name in ((1, "start"), (2, "prev grid done"), (3, "ticket"), (4, "unit landed"), (5, "published"),
                       (6, "prefix known"), (7, "decoded"), (8, "done")):
        # k-th occurrence per warp
        for k in range(4):
            ts = [[t for t, c in e if c == code][k] - t0 for e in ev if len([1 for t, c in e if c == code]) > k]
            if not ts: break
            ts = np.array(ts) / 1e3
            print(f"  {name:15s} #{k}: n={ts.size:5d}  min {ts.min():6.1f}  p10 {np.percentile(ts,10):6.1f}  p50 {np.percentile(ts,50):6.1f}  p90 {np.percentile(ts,90):6.1f}  max {ts.max():6.1f} us")
    # the slowest warps, event by event (code 9: the unit taken)
    order = sorted(range(len(ev)), key=lambda i: -max(t for t, c in ev[i] if c != 9))[:4]
    for i in order:
        print("  slow warp:", " ".join((f"u={t}" if c == 9 else f"{c}@{(t - t0) / 1e3:.1f}") for t, c in ev[i]))
    # the warps whose first publication is the latest (every later unit's prefix waits for them)
    def first_pub(e):
        return next((t for t, c in e if c == 5), 0)
    for i in sorted(range(len(ev)), key=lambda i: -first_pub(ev[i]))[:6]:
        print(f"  late first publication (warp row {i}):", " ".join((f"u={t}" if c == 9 else f"{c}@{(t - t0) / 1e3:.1f}") for t, c in ev[i][:8]))
