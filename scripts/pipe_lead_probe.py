"""Host drop-in (pipelined H2D / decode / D2H) time per call on a config at
several first-chunk sizes.  (It was written for an experimental MVB_PIPE_LEAD
knob -- input chunks queued only a few chunks ahead of the output -- that made
no difference and was removed; the env variable is now only echoed.)"""
import ctypes, os, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1503_07387_b200 import _lib, workload as W

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = {"c2": W.config2, "c1": W.config1, "all1": lambda: W.config5("all1"), "c4s": lambda: W.config4(n=1 << 26)}[name]()
h_in = torch.from_numpy(w.encoded).pin_memory()
h_out = torch.empty(w.count, dtype=torch.int32).pin_memory()
torch.cuda.init()
L = _lib.lib(); res = _lib.MvbResult()
exp = w.expected()
def call():
    rc = (L.mvb_decode_delta_stream(h_in.data_ptr(), w.encoded.size, w.count, w.prev, h_out.data_ptr(), 0, ctypes.byref(res))
          if w.delta else L.mvb_decode_stream(h_in.data_ptr(), w.encoded.size, w.count, h_out.data_ptr(), 0, ctypes.byref(res)))
    assert rc == 0, rc
for chunk in (512 << 10, 1 << 20, 2 << 20):
    _lib.set_host_pipeline(4 << 20, chunk, True)
    call()
    assert np.array_equal(h_out.numpy().view(np.uint32), exp)
    ts = []
    for _ in range(25):
        t = time.perf_counter(); call(); ts.append(time.perf_counter() - t)
    t = float(np.median(ts[3:]))
    print(f"{name} lead={os.environ.get('MVB_PIPE_LEAD', '0')} chunk={chunk >> 10} KiB: {t * 1e3:.3f} ms "
          f"{w.count / t / 1e9:.2f} Gint/s", flush=True)
