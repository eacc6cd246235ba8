"""Batched delta lists through the unit-based kernel (decode_lists.cuh): long
lists whose whole 4 KiB units take the dp2a slices, with everything that makes
a slice hand over to the general range decoder -- integers of 4 and 5 bytes,
malformed runs, count limits, truncation -- at every list alignment.  One
oracle decode per list (the reference's per-list decode_delta_stream loop,
tools/bench/runner.cpp:28-61); bit-exact values and DecodeResults; guard
regions between the lists' outputs stay untouched."""
import numpy as np
import pytest

from paper_1503_07387_b200 import mvb

pytestmark = pytest.mark.gpu

GUARD = 8  # integers of never-written output after every list (an empty list asking for GUARD integers)


def gaps(rng, n, p2=0.15, p3=0.05, p_long=0.0):
    """n gaps: 1-byte by default, 2/3-byte with the given probabilities, 4-5-byte with p_long."""
    u = rng.random(n)
    v = rng.integers(1, 1 << 7, n, dtype=np.uint64)
    two = u < p2
    three = (u >= p2) & (u < p2 + p3)
    lng = u >= 1.0 - p_long
    v[two] = rng.integers(1 << 7, 1 << 14, int(two.sum()), dtype=np.uint64)
    v[three] = rng.integers(1 << 14, 1 << 21, int(three.sum()), dtype=np.uint64)
    v[lng] = rng.integers(1 << 21, 1 << 32, int(lng.sum()), dtype=np.uint64)
    return v.astype(np.uint32)


def run_batch(cuda, oracle, specs, lead):
    """specs: list of (bytes, count, prev).  Every list is followed by an empty
    list of GUARD integers (nothing may be written there)."""
    import torch

    parts, counts, prevs = [], [], []
    for e, cnt, pv in specs:
        parts += [e, np.zeros(0, np.uint8)]
        counts += [cnt, GUARD]
        prevs += [pv, 0]
    byte_off = np.zeros(len(parts) + 1, np.uint64)
    byte_off[1:] = np.cumsum([p.size for p in parts])
    byte_off += lead
    int_off = np.zeros(len(parts) + 1, np.uint64)
    int_off[1:] = np.cumsum(counts)
    data = np.concatenate([np.full(lead, 0x85, np.uint8)] + parts + [np.full(5, 0x85, np.uint8)])
    src = torch.from_numpy(data).to(cuda)
    out = torch.full((int(int_off[-1]) + 4,), -1, dtype=torch.int32, device=cuda)
    res = torch.zeros(len(parts) * 3, dtype=torch.int64, device=cuda)
    order = np.argsort(-np.diff(byte_off).astype(np.int64), kind="stable").astype(np.uint32)
    d = mvb.Decoder(cuda, 1 << 16)
    d.decode_lists(src[:data.size - 5], torch.from_numpy(byte_off.view(np.int64)).to(cuda),
                   torch.from_numpy(int_off.view(np.int64)).to(cuda), out,
                   prev=torch.from_numpy(np.array(prevs, np.uint32).view(np.int32)).to(cuda),
                   order=torch.from_numpy(order.view(np.int32)).to(cuda), results=res, delta=True)
    got = out.cpu().numpy().view(np.uint32)
    rr = res.cpu().numpy().reshape(-1, 3)
    for l in range(0, len(parts), 2):
        span = data[int(byte_off[l]):int(byte_off[l + 1])]
        ro, oo = oracle.decode_delta(span, counts[l], prevs[l])
        assert tuple(int(x) for x in rr[l]) == tuple(ro), (l // 2, rr[l], ro, span.size)
        k = ro[1]
        i0 = int(int_off[l])
        np.testing.assert_array_equal(got[i0:i0 + k], oo[:k], err_msg=f"list {l // 2}")
        # nothing past out + count (mvb_cuda.h: after a failure out[values_written, count) is
        # unspecified): the guard after the list is untouched
        assert (got[i0 + counts[l]:int(int_off[l + 2])] == 0xFFFFFFFF).all(), f"list {l // 2}: stores past count"
        assert tuple(int(x) for x in rr[l + 1]) == (1, 0, 0)  # the guard list: truncated, nothing written
    assert (got[int(int_off[-1]):] == 0xFFFFFFFF).all()


@pytest.mark.parametrize("lead", [0, 1, 7, 15, 16, 29])
def test_long_lists_every_hand_over(cuda, oracle, lead):
    rng = np.random.default_rng(1000 + lead)
    specs = []
    for l in range(120):
        kind = l % 12
        n = int(rng.integers(3000, 40000)) if l % 3 else int(rng.integers(0, 6000))
        p_long = 0.0 if kind < 6 else (0.0005 if kind < 9 else 0.02)
        v = gaps(rng, n, p_long=p_long) if n else np.zeros(0, np.uint32)
        e = oracle.encode_sequence(v) if n else np.zeros(0, np.uint8)
        cnt = n
        if kind == 1 and n > 10:
            cnt = int(rng.integers(1, n))          # count limit somewhere inside
        if kind == 2 and n > 10:
            cnt = n - int(rng.integers(1, 4))      # ... just before the end
        if kind == 3 and e.size > 10:
            e = e[:e.size - int(rng.integers(1, 3))]  # truncated (maybe mid-integer)
            cnt = n + 3
        if kind == 4 and e.size > 100:
            e = e.copy()
            p = int(rng.integers(0, e.size - 8))
            e[p:p + 6] = 0x80                         # over-long run: malformed
        if kind == 5 and e.size > 100:
            e = e.copy()
            p = int(rng.integers(0, e.size - 8))
            e[p:p + 4] = 0x81
            e[p + 4] = 0x10 + int(rng.integers(0, 0x70))  # fifth byte >= 0x10: malformed
        specs.append((e, cnt, int(rng.integers(0, 1 << 32))))
    run_batch(cuda, oracle, specs, lead)


def test_lists_at_unit_multiples(cuda, oracle):
    """All-1-byte lists whose byte length sits at and around multiples of the
    992-byte slice and the four-slice unit (no tail / one-byte tail / count-1
    at a slice's last byte), at alignments 0..15, exact and short counts,
    truncated by one byte."""
    rng = np.random.default_rng(5)
    specs = []
    for k in (1, 3, 4, 5, 8, 9):  # (slices of 992 bytes, units of four slices)
        for d in (-17, -16, -1, 0, 1, 15, 16, 17):
            n = 992 * k + d
            v = rng.integers(0, 1 << 7, n, dtype=np.uint64).astype(np.uint32)
            e = oracle.encode_sequence(v)
            specs.append((e, n, 5))
            specs.append((e, n - 1, 6))
            specs.append((e, n + 2, 7))          # truncated: fewer integers than asked for
            e2 = e.copy()
            e2[-1] |= 0x80                        # the last integer never ends
            specs.append((e2, n, 8))
    for lead in (0, 3, 9):
        run_batch(cuda, oracle, specs, lead)


def test_three_byte_and_long_integers_across_unit_and_slice_seams(cuda, oracle):
    """Integers of 3, 4 and 5 bytes placed so that they straddle every d3 slice
    start (992 i) and the unit boundary of 1-byte streams."""
    rng = np.random.default_rng(9)
    specs = []
    for length in (2, 3, 4, 5):
        lo = 1 << (7 * (length - 1))
        hi = min(1 << (7 * length), 1 << 32)
        for seam in (992, 1984, 2976, 3968, 7936):
            for shift in range(-20, 3):
                n_before = seam + shift + (16 - 3)  # (3 lead bytes in run_batch below)
                v = np.concatenate([rng.integers(0, 1 << 7, n_before, dtype=np.uint64),
                                    rng.integers(lo, hi, 1, dtype=np.uint64),
                                    rng.integers(0, 1 << 7, 9000 - n_before, dtype=np.uint64)]).astype(np.uint32)
                specs.append((oracle.encode_sequence(v), v.size, int(rng.integers(0, 1 << 32))))
    run_batch(cuda, oracle, specs, 3)


def test_offset_validation_follows_tensor_identity_and_version(cuda, oracle):
    """Decoder.decode_lists validates the offset tensors once per tensor object
    and version: a new tensor at a reused address is validated again, and an
    in-place change to decreasing offsets is caught."""
    import torch

    d = mvb.Decoder(cuda, 1 << 16)
    rng = np.random.default_rng(3)
    for n_each in (10, 500, 20):  # same number of lists, different totals; freed tensors' addresses get reused
        vals = [gaps(rng, n_each) for _ in range(4)]
        parts = [oracle.encode_sequence(v) for v in vals]
        bo = np.zeros(5, np.int64)
        bo[1:] = np.cumsum([p.size for p in parts])
        io = np.zeros(5, np.int64)
        io[1:] = np.cumsum([n_each] * 4)
        src = torch.from_numpy(np.concatenate(parts)).to(cuda)
        out = torch.zeros(4 * n_each, dtype=torch.int32, device=cuda)
        d.decode_lists(src, torch.from_numpy(bo).to(cuda), torch.from_numpy(io).to(cuda), out, delta=True)
        want = np.concatenate([np.cumsum(v, dtype=np.uint32) for v in vals])
        np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32), want)
    t_bo, t_io = torch.from_numpy(bo).to(cuda), torch.from_numpy(io).to(cuda)
    d.decode_lists(src, t_bo, t_io, out, delta=True)
    d.decode_lists(src, t_bo, t_io, out, delta=True)  # (cached)
    t_io[2] = 1  # decreasing now
    with pytest.raises(mvb.MvbError):
        d.decode_lists(src, t_bo, t_io, out, delta=True)
