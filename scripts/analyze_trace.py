"""Per-tile timeline summary (see scripts/trace_tiles.py for the slots)."""
import sys

import numpy as np

slots = {0: "start", 1: "count_pub", 3: "phase2_done", 4: "sum_pub", 5: "lookback_done", 6: "stored"}
for cfg in sys.argv[1:]:
    t = np.load(f"gpurun_out/trace_{cfg}.npy").reshape(-1, 8).astype(np.int64)
    t = t[t[:, 0] > 0]
    T0 = t[:, 0].min()
    print(cfg, "tiles", len(t), "span us %.1f" % ((t[:, 6].max() - T0) / 1e3))
    prev = 0
    for k in (1, 3, 4, 5, 6):
        if not (t[:, k] > 0).any():
            continue
        d = (t[:, k] - t[:, prev]) / 1e3
        print(f"  {slots[prev]:>13s} -> {slots[k]:13s} mean {d.mean():6.2f} us p50 {np.median(d):6.2f} p90 {np.percentile(d, 90):6.2f}")
        prev = k
    life = (t[:, 6] - t[:, 0]) / 1e3
    print("  lifetime mean %.2f p50 %.2f" % (life.mean(), np.median(life)))
