"""Randomised parity stress of the host-pointer drop-ins (mvb_decode_stream / mvb_decode_delta_stream,
pipelined chunks from 4 MB on) against the oracle: python scripts/r2/stress_host.py SECONDS [SEED]"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from oracle import Oracle, STRICT, PERMISSIVE
from paper_1503_07387_b200 import mvb

orc = Oracle()
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
t0 = time.time()
cases = fails = 0
while time.time() - t0 < budget:
    n = int(rng.choice([0, 100, 50000, 3_000_000, 6_000_000, 12_000_000])) + int(rng.integers(0, 5000))
    kind = int(rng.integers(0, 3))
    v = rng.integers(0, 1 << 7, n, dtype=np.uint64)
    u = rng.random(n)
    if kind >= 1:
        v[u < 0.3] = rng.integers(1 << 7, 1 << 14, int((u < 0.3).sum()), dtype=np.uint64)
    if kind == 2:
        v[u < 0.05] = rng.integers(1 << 14, 1 << 32, int((u < 0.05).sum()), dtype=np.uint64)
    data = orc.encode_sequence(v.astype(np.uint32)) if n else np.zeros(0, np.uint8)
    count, r = n, rng.random()
    if r < 0.15 and n > 2:
        count = int(rng.integers(1, n))
    elif r < 0.3 and data.size > 3:
        data = data[:data.size - int(rng.integers(1, 4))]
    elif r < 0.4 and data.size > 20:
        data = data.copy()
        p = int(rng.integers(0, data.size - 8))
        data[p:p + 6] = 0x80
    delta = bool(rng.integers(0, 2))
    mode = PERMISSIVE if rng.random() < 0.1 else STRICT
    out = np.full(count + 2, 0xFFFFFFFF, np.uint32)
    if delta:
        res = mvb.decode_delta_stream(data, count, 99, out[:max(count, 1)] if count else out[:0], mvb.DecodeOptions(mode=mode))
        want_r, want = orc.decode_delta(data, count, 99, mode)
    else:
        res = mvb.decode_stream(data, count, out[:max(count, 1)] if count else out[:0], mvb.DecodeOptions(mode=mode))
        want_r, want = orc.decode(data, count, mode)
    got_r = (int(res.status), res.values_written, res.bytes_consumed)
    k = want_r[1]
    ok = got_r == tuple(want_r) and np.array_equal(out[:k], want[:k]) and (out[count:] == 0xFFFFFFFF).all()
    cases += 1
    if not ok:
        fails += 1
        print("MISMATCH", dict(n=n, bytes=int(data.size), count=count, delta=delta, mode=mode, kind=kind), got_r, want_r, flush=True)
print(f"stress_host: {cases} cases, {fails} mismatches, {time.time() - t0:.0f} s")
sys.exit(1 if fails else 0)
