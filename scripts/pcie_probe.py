"""PCIe probe: pinned H2D / D2H bandwidth alone and concurrent, and the
pipelined host drop-in on c2 at several chunk sizes."""
import ctypes, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1503_07387_b200 import _lib, workload as W

dev = torch.device("cuda", 0)
w = W.config2() if len(sys.argv) < 2 else {"c1": W.config1, "all5": lambda: W.config5("all5"), "all1": lambda: W.config5("all1")}[sys.argv[1]]()
n_in, n_out = w.encoded.size, 4 * w.count
h_in = torch.from_numpy(w.encoded).pin_memory()
h_out = torch.empty(w.count, dtype=torch.int32).pin_memory()
d_in = torch.empty(n_in, dtype=torch.uint8, device=dev)
d_out = torch.empty(w.count, dtype=torch.int32, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

def timeit(fn, reps=20):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps

def h2d():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
def both():
    h2d(); d2h()
t1, t2, t3 = timeit(h2d), timeit(d2h), timeit(both)
print(f"H2D {n_in/1e6:.1f} MB {t1*1e6:.0f} us {n_in/t1/1e9:.1f} GB/s; D2H {n_out/1e6:.1f} MB {t2*1e6:.0f} us "
      f"{n_out/t2/1e9:.1f} GB/s; concurrent {t3*1e6:.0f} us")
L = _lib.lib(); res = _lib.MvbResult()
def call():
    rc = (L.mvb_decode_delta_stream(h_in.data_ptr(), n_in, w.count, w.prev, h_out.data_ptr(), 0, ctypes.byref(res)) if w.delta
          else L.mvb_decode_stream(h_in.data_ptr(), n_in, w.count, h_out.data_ptr(), 0, ctypes.byref(res)))
    assert rc == 0
for chunk, grow in ((512 << 10, True), (1 << 20, True), (2 << 20, True), (1 << 20, False)):
    _lib.set_host_pipeline(4 << 20, chunk, grow)
    t = timeit(call, 30)
    print(f"pipelined first chunk {chunk >> 10} KiB grow {grow}: {t*1e6:.0f} us  {w.count/t/1e9:.2f} Gint/s")
_lib.set_host_pipeline(1 << 40)
t = timeit(call, 30)
print(f"unpipelined: {t*1e6:.0f} us  {w.count/t/1e9:.2f} Gint/s")
assert np.array_equal(h_out.numpy().view(np.uint32), w.expected())

_lib.set_host_pipeline()
call()
f = L.mvbx_host_timeline
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
t = (ctypes.c_float * 256)()
n = f(t, 64)
print("chunk  h2d_end  k_start  dec_end  d2h_end (ms)")
for k in range(n):
    print(f"{k:3d} {t[4*k]:8.3f} {t[4*k+1]:8.3f} {t[4*k+2]:8.3f} {t[4*k+3]:8.3f}")
