"""Sharded delta decode of c4 on one GPU, rank r of W: time the totals pass and
the decode pass (and, for comparison, the single-pass decode of the same
shard).  Run under ncu for the DRAM bytes of each pass:
python scripts/r2/shard_traffic.py W r"""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1503_07387_b200 import _lib, mvb, workload as W
world, rank = int(sys.argv[1]), int(sys.argv[2])
w = W.config4()
L = _lib.lib()
cuts = np.zeros(world + 1, np.uint64)
L.mvb_shard_cuts(w.encoded.ctypes.data, w.encoded.size, world, cuts.ctypes.data)
lo, hi = int(cuts[rank]), int(cuts[rank + 1])
dev = torch.device("cuda", 0)
src = torch.from_numpy(np.ascontiguousarray(w.encoded[lo:hi])).to(dev)
n = src.numel()
out = torch.empty(n, dtype=torch.int32, device=dev)
d = mvb.Decoder(dev, capacity_bytes=n)
rec = torch.zeros(2, dtype=torch.int64, device=dev)
carry = torch.zeros(1, dtype=torch.int32, device=dev)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
def two_pass():
    assert L.mvb_delta_totals_device(src.data_ptr(), n, rec.data_ptr(), d.ws.data_ptr(), d.ws_bytes, s) == 0
    assert L.mvb_decode_delta_totaled_device(src.data_ptr(), n, n, 0, carry.data_ptr(), out.data_ptr(),
                                             d.res.data_ptr(), d.ws.data_ptr(), d.ws_bytes, s) == 0
def one_pass():
    d.decode_delta(src, n, 0, out)
for f in (two_pass, one_pass):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): f()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    ints = int(rec[0].item()) if f is two_pass else d.result().values_written
    print(f"W={world} r={rank} {f.__name__}: shard {n/1e6:.0f} MB, {ints} ints, {ms*1e3:.1f} us, "
          f"{ints/ms/1e6:.1f} Gint/s, alg {(n + 4*ints)/ms/1e6:.0f} GB/s", flush=True)
