"""Slices per lane-local path (path-stats build: MVB_CUDA_LIB=build_variants/stats.so)."""
import ctypes, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1503_07387_b200 import _lib, mvb, workload as W
mk = {"c2": W.config2, "c1": W.config1, "c4s": lambda: W.config4(n=1 << 27), "p50d": lambda: W.config5("p50", delta=True),
      "all1": lambda: W.config5("all1"), "all5": lambda: W.config5("all5")}
L = _lib.lib(); f = L.mvbx_path_counts; f.argtypes = [ctypes.c_void_p]
dev = torch.device("cuda", 0)
for name in sys.argv[1:]:
    if name == "c3":
        w = W.config3()
        d = mvb.Decoder(dev, 1 << 16)
        src = torch.from_numpy(w.encoded).to(dev); out = torch.empty(w.count, dtype=torch.int32, device=dev)
        c = (ctypes.c_ulonglong * 4)(); f(c)
        d.decode_lists(src, torch.from_numpy(w.byte_offsets.astype(np.uint64).view(np.int64)).to(dev),
                       torch.from_numpy(w.int_offsets.astype(np.uint64).view(np.int64)).to(dev), out, delta=True)
        torch.cuda.synchronize(); f(c); tot = sum(c)
        print(f"c3    slices {tot}: 2-byte {c[0]/tot:.3f} fast {c[1]/tot:.3f} general-interior {c[2]/tot:.3f} edge {c[3]/tot:.3f}")
        continue
    w = mk[name]()
    src = torch.from_numpy(w.encoded).to(dev); out = torch.empty(w.count, dtype=torch.int32, device=dev)
    d = mvb.Decoder(dev, w.encoded.size)
    c = (ctypes.c_ulonglong * 4)(); f(c)
    if w.delta: d.decode_delta(src, w.count, w.prev, out)
    else: d.decode(src, w.count, out)
    torch.cuda.synchronize(); f(c)
    tot = sum(c)
    print(f"{name:5s} slices {tot}: 2-byte {c[0]/tot:.3f} fast {c[1]/tot:.3f} general-interior {c[2]/tot:.3f} edge {c[3]/tot:.3f}")
