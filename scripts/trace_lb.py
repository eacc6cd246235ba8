"""CTA-pipelined kernel (traced): does barrier #1 of iteration i wait for the
lookback of t_{i-2}?  Compares lookback-done(t_{i-2}) with count-publish(t_i)
(which follows barrier #1)."""
import sys
import numpy as np

t = np.load(sys.argv[1]).reshape(-1, 8).astype(np.int64)
n = len(t)
G = int(sys.argv[2])
ok = t[:, 0] > 0
lb_done = t[:, 5]
cnt_pub = t[:, 1]
ph2 = t[:, 3]
d_wait = []
for x in range(2 * G, n):
    if ok[x] and ok[x - 2 * G] and lb_done[x - 2 * G] > 0:
        d_wait.append((cnt_pub[x] - lb_done[x - 2 * G]) / 1e3)
d = np.array(d_wait)
print("count_pub(t_i) - lookback_done(t_{i-2}) us: mean %.2f p10 %.2f p50 %.2f p90 %.2f; frac<0.1us %.2f"
      % (d.mean(), np.percentile(d, 10), np.median(d), np.percentile(d, 90), np.mean(d < 0.1)))
it = (t[G:, 0] - t[:-G, 0])[ok[G:] & ok[:-G]] / 1e3
print("iteration time us: mean %.2f p50 %.2f p90 %.2f" % (it.mean(), np.median(it), np.percentile(it, 90)))
