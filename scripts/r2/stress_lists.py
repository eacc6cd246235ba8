"""Randomised parity stress of the batched delta lists kernel against one oracle decode per list
(run on the GPU box): random batches, list lengths 0..20000 integers of short / mixed / long codes,
count limits, truncation, over-long runs, fifth bytes >= 0x10, random batch misalignment.
python scripts/r2/stress_lists.py SECONDS [SEED]"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from oracle import Oracle
from paper_1503_07387_b200 import mvb

orc = Oracle()
dev = torch.device("cuda", 0)
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
d = mvb.Decoder(dev, 1 << 16)
t0 = time.time()
n_lists_total = fails = batches = 0


def gaps(n, kind):
    v = rng.integers(1, 1 << 7, n, dtype=np.uint64)
    u = rng.random(n)
    if kind >= 1:
        v[u < 0.15] = rng.integers(1 << 7, 1 << 14, int((u < 0.15).sum()), dtype=np.uint64)
        v[u < 0.03] = rng.integers(1 << 14, 1 << 21, int((u < 0.03).sum()), dtype=np.uint64)
    if kind >= 2:
        p = 0.001 if kind == 2 else 0.3
        v[u > 1 - p] = rng.integers(1 << 21, 1 << 32, int((u > 1 - p).sum()), dtype=np.uint64)
    return v.astype(np.uint32)


while time.time() - t0 < budget:
    parts, counts, prevs = [], [], []
    for _ in range(int(rng.integers(20, 200))):
        n = int(rng.choice([0, 1, 15, 200, 992, 3968, 7936])) + int(rng.integers(0, 30)) if rng.random() < 0.5 else int(rng.integers(0, 20000))
        e = orc.encode_sequence(gaps(n, int(rng.integers(0, 4)))) if n else np.zeros(0, np.uint8)
        cnt, r = n, rng.random()
        if r < 0.1 and n > 2:
            cnt = int(rng.integers(1, n))
        elif r < 0.2 and e.size > 3:
            e = e[:e.size - int(rng.integers(1, 4))]
            cnt = n + int(rng.integers(0, 3))
        elif r < 0.27 and e.size > 20:
            e = e.copy()
            p = int(rng.integers(0, e.size - 8))
            e[p:p + int(rng.integers(5, 8))] = 0x80
        elif r < 0.32 and e.size > 20:
            e = e.copy()
            p = int(rng.integers(0, e.size - 8))
            e[p:p + 4] = 0x81
            e[p + 4] = 0x10 + int(rng.integers(0, 0x70))
        parts += [e, np.zeros(0, np.uint8)]
        counts += [cnt, 4]  # (a guard list of 4 never-written integers after every list)
        prevs += [int(rng.integers(0, 1 << 32)), 0]
    lead = int(rng.integers(0, 16))
    byte_off = np.zeros(len(parts) + 1, np.uint64)
    byte_off[1:] = np.cumsum([p.size for p in parts])
    int_off = np.zeros(len(parts) + 1, np.uint64)
    int_off[1:] = np.cumsum(counts)
    data = np.concatenate([np.full(16, 0x85, np.uint8)] + parts + [np.full(5, 0x85, np.uint8)])
    src = torch.from_numpy(data).to(dev)[16 - lead:]  # the batch starts `lead` bytes before a 16-byte boundary... then at one
    byte_off += lead
    out = torch.full((int(int_off[-1]) + 4,), -1, dtype=torch.int32, device=dev)
    res = torch.zeros(len(parts) * 3, dtype=torch.int64, device=dev)
    order = np.argsort(-np.diff(byte_off).astype(np.int64), kind="stable").astype(np.uint32)
    d.decode_lists(src[:data.size - 16 + lead - 5], torch.from_numpy(byte_off.view(np.int64)).to(dev),
                   torch.from_numpy(int_off.view(np.int64)).to(dev), out,
                   prev=torch.from_numpy(np.array(prevs, np.uint32).view(np.int32)).to(dev),
                   order=torch.from_numpy(order.view(np.int32)).to(dev) if rng.random() < 0.7 else None, results=res, delta=True)
    got = out.cpu().numpy().view(np.uint32)
    rr = res.cpu().numpy().reshape(-1, 3)
    hdata = data[16 - lead:]
    for l in range(0, len(parts), 2):
        span = hdata[int(byte_off[l]):int(byte_off[l + 1])]
        ro, oo = orc.decode_delta(span, counts[l], prevs[l])
        i0, k = int(int_off[l]), ro[1]
        ok = tuple(int(x) for x in rr[l]) == tuple(ro) and np.array_equal(got[i0:i0 + k], oo[:k]) and \
            (got[i0 + counts[l]:int(int_off[l + 2])] == 0xFFFFFFFF).all()
        n_lists_total += 1
        if not ok:
            fails += 1
            print("MISMATCH list", l // 2, "bytes", span.size, "count", counts[l], tuple(int(x) for x in rr[l]), ro, flush=True)
    batches += 1
print(f"stress_lists: {batches} batches, {n_lists_total} lists, {fails} mismatches, {time.time() - t0:.0f} s")
sys.exit(1 if fails else 0)
