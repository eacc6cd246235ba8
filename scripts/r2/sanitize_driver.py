"""Small decodes through every kernel family, for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck): the fused single-read decoder
(plain, delta, its totals-only and decode-only passes), the two-kernel
segmented pair (the pipelined host drop-in's chunks), the batched-lists
kernel, the per-tile permissive kernel, the device encoder.  Exits non-zero on
any mismatch with the oracle."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from oracle import Oracle, PERMISSIVE, STRICT
from paper_1503_07387_b200 import _lib, mvb, workload as W

orc = Oracle()
dev = torch.device("cuda", 0)
L = _lib.lib()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300000
fails = 0


def check(tag, got, want):
    global fails
    if not got == want:
        print("MISMATCH", tag, got, want, flush=True)
        fails += 1


v = W.mixed_values(n, 5)
enc = orc.encode_sequence(v)
g = W.mixture(n, 6, 0.4, (1, 127), (128, 70000))
encg = orc.encode_sequence(g)
d = mvb.Decoder(dev, capacity_bytes=int(max(enc.size, encg.size)))
for data, vals, delta in ((enc, v, False), (encg, g, True)):
    src = torch.from_numpy(data).to(dev)
    for mode in (STRICT, PERMISSIVE):
        for choice in ((0, 6) if mode == STRICT else (0,)):
            _lib.set_kernel_choice(choice)
            out = torch.empty(vals.size, dtype=torch.int32, device=dev)
            if delta:
                d.decode_delta(src, vals.size, 9, out, mode)
                ro, oo = orc.decode_delta(data, vals.size, 9, mode)
            else:
                d.decode(src, vals.size, out, mode)
                ro, oo = orc.decode(data, vals.size, mode)
            r = d.result()
            check(f"stream delta={delta} mode={mode} choice={choice}", ((int(r.status), r.values_written, r.bytes_consumed),
                                                                       bool(np.array_equal(out.cpu().numpy().view(np.uint32), oo))), (tuple(ro), True))
    _lib.set_kernel_choice(0)
# totals-only + decode-only passes (sharded building blocks)
src = torch.from_numpy(encg).to(dev)
rec = torch.zeros(2, dtype=torch.int64, device=dev)
out = torch.empty(g.size, dtype=torch.int32, device=dev)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
assert L.mvb_delta_totals_device(src.data_ptr(), encg.size, rec.data_ptr(), d.ws.data_ptr(), d.ws_bytes, s) == 0
assert L.mvb_decode_delta_totaled_device(src.data_ptr(), encg.size, g.size, 4, None, out.data_ptr(), d.res.data_ptr(),
                                         d.ws.data_ptr(), d.ws_bytes, s) == 0
ro, oo = orc.decode_delta(encg, g.size, 4)
r = d.result()
check("totals+totaled", ((int(r.status), r.values_written, r.bytes_consumed), bool(np.array_equal(out.cpu().numpy().view(np.uint32), oo)),
                         rec.cpu().tolist()[0]), (tuple(ro), True, g.size))
# host pipelined drop-in on small chunks (the segmented pair over chunks)
_lib.set_host_pipeline(1 << 16, 1 << 14, True)
o = np.zeros(g.size, np.uint32)
r = mvb.decode_delta_stream(encg, g.size, 4, o)
check("host pipelined", ((int(r.status), r.values_written, r.bytes_consumed), bool(np.array_equal(o, oo))), (tuple(ro), True))
_lib.set_host_pipeline()
# batched lists
parts, counts = [], []
rng = np.random.default_rng(3)
for l in range(300):
    k = int(rng.integers(0, 2000))
    x = W.mixed_values(k, l + 1) if k else np.zeros(0, np.uint32)
    parts.append(orc.encode_sequence(x) if k else np.zeros(0, np.uint8))
    counts.append(k)
bo = np.zeros(len(parts) + 1, np.uint64); bo[1:] = np.cumsum([p.size for p in parts])
io = np.zeros(len(parts) + 1, np.uint64); io[1:] = np.cumsum(counts)
data = np.concatenate(parts)
outl = torch.zeros(int(io[-1]) + 1, dtype=torch.int32, device=dev)
res = torch.zeros(3 * len(parts), dtype=torch.int64, device=dev)
d.decode_lists(torch.from_numpy(data).to(dev), torch.from_numpy(bo.view(np.int64)).to(dev),
               torch.from_numpy(io.view(np.int64)).to(dev), outl, results=res, delta=True)
got = outl.cpu().numpy().view(np.uint32)
ok = True
for l, p in enumerate(parts):
    rl, ol = orc.decode_delta(p, counts[l], 0)
    ok &= np.array_equal(got[int(io[l]):int(io[l + 1])], ol[:counts[l]])
check("lists", ok, True)
# device encoder
enc_d = mvb.encode_device(torch.from_numpy(v).to(dev))
check("encoder", bool(np.array_equal(enc_d.cpu().numpy(), enc)), True)
print("sanitize driver done, mismatches:", fails, flush=True)
sys.exit(1 if fails else 0)
