"""Per-tile timeline of one decode (profiling aid).

    python scripts/trace_tiles.py <cfg> [tag]      (MVB_CUDA_LIB selects a variant library)

Writes gpurun_out/trace_<cfg>[_tag].npy: 8 u64 per tile (%globaltimer ns):
start, count published, count lookback done, phase 2 done, sum aggregate,
sum lookback done, end, smid<<32|blockIdx.  Also prints the untraced kernel
time (CUDA events, L2 flushed before each launch)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1503_07387_b200 import _lib, mvb, workload as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
tag = ("_" + sys.argv[2]) if len(sys.argv) > 2 else ""
w = {"c1": W.config1, "c2": W.config2, "all1": lambda: W.config5("all1"), "all5": lambda: W.config5("all5")}[cfg]()
dev = torch.device("cuda", 0)
L = _lib.lib()
if os.environ.get("MVB_KERNEL"):  # strict kernel variant to trace (3 = warp-sliced v3)
    _lib.set_kernel_choice(int(os.environ["MVB_KERNEL"]))
L.mvbx_decode_traced.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint32,
                                 ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                 ctypes.c_void_p, ctypes.c_void_p]
src = torch.from_numpy(w.encoded).to(dev)
out = torch.empty(w.count, dtype=torch.int32, device=dev)
d = mvb.Decoder(dev, w.encoded.size)
tiles = (w.encoded.size + 4095) // 4096 + 1
trace = torch.zeros(tiles * 8, dtype=torch.int64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
times = []
for it in range(8):
    flush.fill_(it)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    if w.delta:
        d.decode_delta(src, w.count, w.prev, out)
    else:
        d.decode(src, w.count, out)
    e.record()
    torch.cuda.synchronize()
    times.append(s.elapsed_time(e) * 1e3)
expected = torch.from_numpy(w.expected().view(np.int32)).to(dev)
assert torch.equal(out, expected), "mismatch"
print("grid", L.mvbx_last_grid() if hasattr(L, "mvbx_last_grid") else "?")
for it in range(3):
    flush.fill_(it)
    torch.cuda.synchronize()
    rc = L.mvbx_decode_traced(src.data_ptr(), w.encoded.size, w.count, int(w.delta), w.prev, out.data_ptr(), 0,
                              d.res.data_ptr(), d.ws.data_ptr(), d.ws_bytes,
                              torch.cuda.current_stream().cuda_stream, trace.data_ptr())
    assert rc == 0
    torch.cuda.synchronize()
r = d.result()
assert r.values_written == w.count
os.makedirs("gpurun_out", exist_ok=True)
np.save(f"gpurun_out/trace_{cfg}{tag}.npy", trace.cpu().numpy())
print(f"{cfg}{tag}: kernel us median {np.median(times[2:]):.1f} min {min(times[2:]):.1f}")
