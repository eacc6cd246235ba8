"""Randomised parity stress of the device decode paths against the oracle (run on the GPU box):
random sizes (including unit / slice multiples +-k), byte-length mixes (short, mixed, uniform 4/5-byte),
input misalignments, plain / delta, count limits, truncation, injected over-long runs.
python scripts/r2/stress.py SECONDS [SEED]"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from oracle import Oracle, STRICT, PERMISSIVE
from paper_1503_07387_b200 import mvb

orc = Oracle()
dev = torch.device("cuda", 0)
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
d = mvb.Decoder(dev, capacity_bytes=1 << 22)
t0 = time.time()
n_cases = fails = 0


def values(n, kind):
    if kind == 0:  # 1-2 bytes
        v = rng.integers(0, 1 << 14, n, dtype=np.uint64)
        v[rng.random(n) < 0.6] &= 0x7F
    elif kind == 1:  # 1-3 bytes, rare longer
        v = rng.integers(0, 1 << 7, n, dtype=np.uint64)
        u = rng.random(n)
        v[u < 0.2] = rng.integers(1 << 7, 1 << 14, int((u < 0.2).sum()), dtype=np.uint64)
        v[u < 0.03] = rng.integers(1 << 14, 1 << 21, int((u < 0.03).sum()), dtype=np.uint64)
        v[u < 0.001] = rng.integers(1 << 21, 1 << 32, int((u < 0.001).sum()), dtype=np.uint64)
    elif kind == 2:  # mixed 1-5
        ln = rng.integers(1, 6, n)
        lo = np.array([0, 0, 1 << 7, 1 << 14, 1 << 21, 1 << 28], np.uint64)[ln]
        hi = np.array([0, 1 << 7, 1 << 14, 1 << 21, 1 << 28, 1 << 32], np.uint64)[ln]
        v = lo + (rng.random(n) * (hi - lo)).astype(np.uint64)
    else:  # uniform 4 or 5 bytes, sometimes one odd integer
        L = 4 if kind == 3 else 5
        v = rng.integers(1 << (7 * (L - 1)), min(1 << (7 * L), 1 << 32), n, dtype=np.uint64)
        if n and rng.random() < 0.3:
            v[rng.integers(0, n)] = rng.integers(0, 1 << 14)
    return v.astype(np.uint32)


while time.time() - t0 < budget:
    base = int(rng.choice([0, 992, 1024, 3968, 4096, 8192, 40960, 200000]))
    n_bytes_target = max(0, base + int(rng.integers(-40, 41))) if rng.random() < 0.7 else int(rng.integers(0, 300000))
    kind = int(rng.integers(0, 5))
    per = [1.4, 1.25, 3.0, 4.0, 5.0][kind]
    n = int(n_bytes_target / per)
    v = values(n, kind)
    data = orc.encode_sequence(v) if n else np.zeros(0, np.uint8)
    count = n
    r = rng.random()
    if r < 0.15 and n > 2:
        count = int(rng.integers(1, n))
    elif r < 0.3 and data.size > 3:
        data = data[:data.size - int(rng.integers(1, 4))]
    elif r < 0.4 and data.size > 20:
        data = data.copy()
        p = int(rng.integers(0, data.size - 8))
        data[p:p + int(rng.integers(5, 8))] = 0x80
    delta = bool(rng.integers(0, 2))
    mode = PERMISSIVE if rng.random() < 0.1 else STRICT
    in_off = int(rng.integers(0, 16))
    src = torch.zeros(data.size + in_off + 16, dtype=torch.uint8, device=dev)
    src[in_off:in_off + data.size] = torch.from_numpy(data.copy()).to(dev)
    out = torch.full((count + 9,), -1, dtype=torch.int32, device=dev)
    inp = src[in_off:in_off + data.size]
    if delta:
        d.decode_delta(inp, count, 12345, out[1:1 + count], mode, in_len=data.size)
        want_r, want = orc.decode_delta(data, count, 12345, mode)
    else:
        d.decode(inp, count, out[1:1 + count], mode, in_len=data.size)
        want_r, want = orc.decode(data, count, mode)
    res = d.result()
    got = out.cpu().numpy().view(np.uint32)
    got_r = (int(res.status), res.values_written, res.bytes_consumed)
    k = want_r[1]
    ok = got_r == tuple(want_r) and np.array_equal(got[1:1 + k], want[:k]) and got[0] == 0xFFFFFFFF and (got[1 + count:] == 0xFFFFFFFF).all()
    n_cases += 1
    if not ok:
        fails += 1
        print("MISMATCH", dict(kind=kind, n=n, bytes=int(data.size), count=count, delta=delta, mode=mode, in_off=in_off), got_r, want_r, flush=True)
print(f"stress: {n_cases} cases, {fails} mismatches, {time.time() - t0:.0f} s")
sys.exit(1 if fails else 0)
