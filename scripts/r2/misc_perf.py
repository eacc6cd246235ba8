"""Timings outside the bench contract, for the record (run on the GPU box):
permissive-mode decodes (the per-tile kernel) of c1 / c2 / c5 P(2B)=.5, and the device encoder
(mvb_encode_sequence_device) on c1's values and on a 2^26 1-2-byte mixture."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1503_07387_b200 import _lib, mvb
import bench

dev = torch.device("cuda", 0)
L = _lib.lib()


def timed(fn, n):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


for cfg in ("c1", "c2", "c5_p50"):
    w = bench.make_workload(cfg)
    src = torch.from_numpy(w.encoded).to(dev)
    out = torch.empty(w.count, dtype=torch.int32, device=dev)
    d = mvb.Decoder(dev, capacity_bytes=int(w.encoded.size))
    exp = torch.from_numpy(w.expected().view(np.int32)).to(dev)
    for mode in (0, 1):
        f = (lambda: d.decode_delta(src, w.count, w.prev, out, mode)) if w.delta else (lambda: d.decode(src, w.count, out, mode))
        f()
        torch.cuda.synchronize()
        ok = torch.equal(out, exp)
        ms = timed(f, 50)
        alg = w.encoded.size + 4 * w.count
        print(f"{cfg} mode={'permissive' if mode else 'strict'} ok={ok} {ms * 1e3:.1f} us {w.count / ms / 1e6:.1f} Gint/s {alg / ms / 1e6:.0f} GB/s", flush=True)

# device encoder
for name, vals in (("c1 values (1-5 bytes)", bench.make_workload("c1").values if hasattr(bench.make_workload("c1"), "values") else None),):
    pass
rng = np.random.default_rng(1)
for name, v in (("2^24 mixed 1-5 bytes", None), ("2^26 1-2 bytes", None)):
    if v is None:
        if "mixed" in name:
            from paper_1503_07387_b200 import workload as W
            v = W.mixed_values(1 << 24, 42)
        else:
            v = rng.integers(0, 1 << 14, 1 << 26, dtype=np.uint64).astype(np.uint32)
            v[rng.random(v.size) < 0.5] &= 0x7F
    t = torch.from_numpy(v.view(np.int32)).to(dev)
    n = int(t.numel())
    ws = torch.empty(max(int(L.mvb_encode_workspace_bytes(n)), 8), dtype=torch.uint8, device=dev)
    outb = torch.empty(5 * n, dtype=torch.uint8, device=dev)
    meta = torch.zeros(2, dtype=torch.int64, device=dev)
    stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    f = lambda: L.mvb_encode_sequence_device(t.data_ptr(), n, outb.data_ptr(), meta.data_ptr(), ws.data_ptr(), ws.numel(), stream)
    ms = timed(f, 20)
    nbytes = int(meta.cpu()[0])
    print(f"device encoder, {name}: {ms * 1e3:.1f} us, {n / ms / 1e6:.1f} Gint/s, {(4 * n + nbytes) / ms / 1e6:.0f} GB/s (in + out)", flush=True)
