"""Debug: decode a config with the default (fused) kernel several times and report mismatches."""
import ctypes, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1503_07387_b200 import _lib, mvb
import bench
cfg = sys.argv[1]
w = bench.make_workload(cfg)
dev = torch.device("cuda", 0)
src = torch.from_numpy(w.encoded).to(dev)
out = torch.empty(w.count, dtype=torch.int32, device=dev)
d = mvb.Decoder(dev, capacity_bytes=int(w.encoded.size))
L = _lib.lib()
has_set = hasattr(L, "mvbx_set_fused")
if has_set:
    L.mvbx_set_fused.argtypes = [ctypes.c_size_t, ctypes.c_longlong]
exp = torch.from_numpy(w.expected().view(np.int32)).to(dev)
for arg in sys.argv[2:]:
    seg, lag = (int(x) for x in arg.split(":"))
    if has_set:
        L.mvbx_set_fused(seg, lag)
    for rep in range(4):
        out.fill_(-1)
        if w.delta: d.decode_delta(src, w.count, w.prev, out)
        else: d.decode(src, w.count, out)
        r = d.result()
        bad = (out != exp).nonzero().flatten()
        nb = bad.numel()
        msg = f"{cfg} seg={seg} lag={lag} rep={rep} result={int(r.status), r.values_written, r.bytes_consumed} mismatches={nb}"
        if nb:
            b = bad.cpu().numpy()
            # contiguous runs
            runs = np.split(b, np.nonzero(np.diff(b) != 1)[0] + 1)
            msg += f" runs={len(runs)} first={[(int(x[0]), int(x[-1]) - int(x[0]) + 1) for x in runs[:6]]}"
            i = int(b[0])
            msg += f" got={out[i:i+4].cpu().numpy().view(np.uint32)} exp={exp[i:i+4].cpu().numpy().view(np.uint32)}"
            dd = (out[b[:8]].to(torch.int64) - exp[b[:8]].to(torch.int64)) & 0xFFFFFFFF
            msg += f" diff={dd.cpu().numpy()}"
        print(msg, flush=True)
