"""Timeline summary of a v3 trace (slots in decode_v3.cuh, MVB_T3)."""
import sys

import numpy as np

names = ["ticket", "p1_start", "p2_done", "published", "lb_start", "resolved", "store"]
for cfg in sys.argv[1:]:
    t = np.load(f"gpurun_out/trace_{cfg}.npy").reshape(-1, 8).astype(np.int64)
    t = t[(t[:, 0] > 0) & (t[:, 6] > 0)]
    T0 = t[:, 0].min()
    print(cfg, "tiles", len(t), "span us %.1f" % ((t[:, 6].max() - T0) / 1e3))
    for a, b in [(0, 1), (1, 2), (2, 3), (2, 4), (4, 5), (5, 6), (2, 6), (3, 5)]:
        d = (t[:, b] - t[:, a]) / 1e3
        print(f"  {names[a]:>10s} -> {names[b]:10s} mean {d.mean():7.2f} p10 {np.percentile(d, 10):7.2f} "
              f"p50 {np.median(d):7.2f} p90 {np.percentile(d, 90):7.2f} max {d.max():7.2f} us")
    # how late is the resolution relative to when the predecessor tile was published?
    order = np.argsort(np.arange(len(t)))
    pub = t[:, 3]
    late = np.maximum.accumulate(pub)  # latest publication among tiles <= i
    d = (t[:, 5] - late) / 1e3
    print(f"  resolved - max(pub of tiles <= t): mean {d.mean():.2f} p50 {np.median(d):.2f} p90 {np.percentile(d, 90):.2f}")
    d = (late - t[:, 3]) / 1e3
    print(f"  max(pub of tiles <= t) - own pub: mean {d.mean():.2f} p50 {np.median(d):.2f} p90 {np.percentile(d, 90):.2f}")
    # per-iteration duration of a CTA (p1_start deltas by block)
    blk = t[:, 7] & 0xFFFFFFFF
    it = []
    for bb in np.unique(blk)[:400]:
        s = np.sort(t[blk == bb, 1])
        it.extend(np.diff(s) / 1e3)
    it = np.array(it)
    print(f"  CTA iteration (p1_start deltas) mean {it.mean():.2f} p50 {np.median(it):.2f} p90 {np.percentile(it, 90):.2f}")
