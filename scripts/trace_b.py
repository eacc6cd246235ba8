"""Kernel B per-warp timeline (trace build: MVB_CUDA_LIB=build_variants/trace.so).
usage: trace_b.py CFG"""
import ctypes, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1503_07387_b200 import _lib, mvb, workload as W
mk = {"c2": W.config2, "c1": W.config1, "p50d": lambda: W.config5("p50", delta=True)}
w = mk[sys.argv[1] if len(sys.argv) > 1 else "c2"]()
dev = torch.device("cuda", 0)
srcs = [torch.from_numpy(w.encoded).to(dev) for _ in range(4)]
out = torch.empty(w.count, dtype=torch.int32, device=dev)
buf = torch.zeros(6 * 200000, dtype=torch.int64, device=dev)
L = _lib.lib()
L.mvbx_set_trace_b.argtypes = [ctypes.c_void_p]
d = mvb.Decoder(dev, w.encoded.size)
def run(k):
    if w.delta: d.decode_delta(srcs[k % 4], w.count, w.prev, out)
    else: d.decode(srcs[k % 4], w.count, out)
for k in range(8): run(k)
torch.cuda.synchronize()
L.mvbx_set_trace_b(buf.data_ptr())
run(9); torch.cuda.synchronize()
L.mvbx_set_trace_b(None)
t = buf.view(-1, 6).cpu().numpy()
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
st, wt, pf, en, nseg = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, (t[:, 3] - t0) / 1e3, t[:, 4]
q = lambda a: " ".join(f"{np.percentile(a, p):7.2f}" for p in (0, 10, 50, 90, 100))
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'c2'}: warps {len(t)}  (us; percentiles 0/10/50/90/100)")
print("start       ", q(st))
print("after wait  ", q(wt))
print("wait dur    ", q(wt - st))
print("prefix dur  ", q(pf - wt))
print("decode dur  ", q(en - pf))
print("end         ", q(en))
print("segs/warp   ", q(nseg.astype(float)))
sm = t[:, 5]
ends = {}
for k in np.unique(sm):
    e = en[sm == k]
    ends[k] = (e.min(), e.max(), (sm == k).sum())
mx = np.array([v[1] for v in ends.values()]); mn = np.array([v[0] for v in ends.values()])
nw = np.array([v[2] for v in ends.values()])
print("per-SM last end ", q(mx))
print("per-SM first end", q(mn))
print("warps per SM    ", q(nw.astype(float)))
k = max(ends, key=lambda x: ends[x][1])
sel = np.where(sm == k)[0]
print(f"slowest SM {k}: warps {sel[:24].tolist()}")
print("  starts", np.round(st[sel], 2).tolist())
print("  ends  ", np.round(en[sel], 2).tolist())
k2 = min(ends, key=lambda x: ends[x][1])
sel2 = np.where(sm == k2)[0]
print(f"fastest SM {k2}: warps {sel2[:24].tolist()}")
order = np.argsort(-en)[:6]
print("latest warps:", [(int(i), round(float(en[i]), 2), round(float(pf[i] - wt[i]), 2), int(sm[i])) for i in order])
