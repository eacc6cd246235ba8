"""Parity of the default lane-local decoder's distinct paths with the oracle:
the fast path (1..4-byte integers, interior slices) against the general path
(5-byte and malformed integers, range edges, the slice holding integer
count-1), the swizzled staging layout of dense (mostly 1-byte) ranges, the
16-byte (delta) and 32-byte (plain) lane widths, and kernel A's digit-weight
segment sums with kernel B's straddle correction at every run start.  All
comparisons bit-exact."""
import numpy as np
import pytest

from oracle import Oracle, STRICT
from paper_1503_07387_b200 import mvb

from test_decode_gpu import dev_decode, gpu_decode

pytestmark = pytest.mark.gpu


def _values_of_lengths(rng, lengths):
    """One value per requested encoded length (1..5 bytes)."""
    lo = np.array([0, 1 << 7, 1 << 14, 1 << 21, 1 << 28], np.uint64)
    hi = np.array([1 << 7, 1 << 14, 1 << 21, 1 << 28, 1 << 32], np.uint64)
    lengths = np.asarray(lengths)
    return (lo[lengths - 1] + (rng.random(lengths.size) * (hi - lo)[lengths - 1]).astype(np.uint64)).astype(np.uint32)


def _blocky_values(n, seed):
    """Runs of 1-byte, 2-byte, 3..4-byte and 5-byte integers of random lengths
    (dense ranges next to sparse ones, fast slices next to general ones)."""
    rng = np.random.default_rng(seed)
    out = []
    total = 0
    while total < n:
        kind = rng.integers(0, 5)
        run = int(rng.integers(1, 4000))
        if kind == 0:
            lens = np.ones(run, np.int64)
        elif kind == 1:
            lens = rng.integers(1, 3, run)
        elif kind == 2:
            lens = rng.integers(3, 5, run)
        elif kind == 3:
            lens = np.full(run, 5)
        else:
            lens = rng.integers(1, 6, run)
        out.append(_values_of_lengths(rng, lens))
        total += run
    return np.concatenate(out)[:n]


@pytest.fixture(scope="module")
def oracle():
    return Oracle()


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_blocky_streams_plain_and_delta(oracle, seed):
    """Dense, sparse and mixed runs back to back: both lane widths, both
    staging layouts, fast and general slices in one decode."""
    v = _blocky_values(1_500_000, seed)
    enc = oracle.encode_sequence(v)
    ro, oo = oracle.decode(enc, v.size)
    r, out = gpu_decode(enc, v.size)
    assert r == ro and np.array_equal(out, oo)
    ro, oo = oracle.decode_delta(enc, v.size, 12345)
    r, out = gpu_decode(enc, v.size, delta=True, prev=12345)
    assert r == ro and np.array_equal(out, oo)


def test_delta_straddles_at_every_run_start(oracle):
    """Only 3..5-byte integers: almost every segment (and so every warp run)
    starts inside an integer, exercising the straddle correction of the
    digit-weight segment sums."""
    rng = np.random.default_rng(7)
    v = _values_of_lengths(rng, rng.integers(3, 6, 2_000_000))
    enc = oracle.encode_sequence(v)
    ro, oo = oracle.decode_delta(enc, v.size, 0xFFFFFFF0)
    r, out = gpu_decode(enc, v.size, delta=True, prev=0xFFFFFFF0)
    assert r == ro and np.array_equal(out, oo)


@pytest.mark.parametrize("delta", [False, True])
def test_count_limits_inside_slices(oracle, delta):
    """count below the stream's integer count, ending at many positions
    inside 512-byte and 1 KiB slices (the general path's end-of-count)."""
    rng = np.random.default_rng(11)
    v = _values_of_lengths(rng, rng.integers(1, 3, 300_000))
    enc = oracle.encode_sequence(v)
    for count in (1, 2, 341, 342, 683, 1023, 1024, 1025, 4099, 150_001, 299_999):
        if delta:
            ro, oo = oracle.decode_delta(enc, count, 5)
            r, out = gpu_decode(enc, count, delta=True, prev=5)
        else:
            ro, oo = oracle.decode(enc, count)
            r, out = gpu_decode(enc, count)
        assert r == ro and np.array_equal(out[: ro[1]], oo[: ro[1]]), (count, delta)


@pytest.mark.parametrize("delta", [False, True])
def test_dense_misaligned_with_guards(oracle, delta):
    """All-1-byte data (swizzled staging) at every input and output
    misalignment, with guard words around the output."""
    import torch

    cuda = torch.device("cuda", 0)
    rng = np.random.default_rng(3)
    v = rng.integers(0, 128, 70_001).astype(np.uint32)
    enc = oracle.encode_sequence(v)
    for in_off, out_off in ((0, 0), (1, 1), (7, 2), (15, 3), (8, 0)):
        if delta:
            ro, oo = oracle.decode_delta(enc, v.size, 99)
        else:
            ro, oo = oracle.decode(enc, v.size)
        r, out = dev_decode(torch, cuda, enc, v.size, STRICT, delta, 99, in_off, out_off)
        assert r == ro and np.array_equal(out, oo), (in_off, out_off, delta)


def test_malformed_inside_dense_and_sparse_runs(oracle):
    """A malformed run injected into dense data and into 5-byte data: the
    first malformed integer's index and position, values before it."""
    rng = np.random.default_rng(5)
    for lens in (np.ones(200_000, np.int64), np.full(60_000, 5), rng.integers(1, 3, 150_000)):
        v = _values_of_lengths(rng, lens)
        enc = oracle.encode_sequence(v)
        for pos in (100, 1023, 1024, 50_001, enc.size - 7):
            bad = enc.copy()
            bad[pos:pos + 6] = 0x80
            for delta in (False, True):
                if delta:
                    ro, oo = oracle.decode_delta(bad, v.size, 1)
                    r, out = gpu_decode(bad, v.size, delta=True, prev=1)
                else:
                    ro, oo = oracle.decode(bad, v.size)
                    r, out = gpu_decode(bad, v.size)
                assert r == ro and np.array_equal(out[: ro[1]], oo[: ro[1]]), (lens[0], pos, delta)


@pytest.mark.parametrize("delta", [False, True])
def test_lists_dense_and_sparse_around_slice_sizes(oracle, delta):
    """Batched lists whose encoded sizes sit around 512 / 1024 / 2048 bytes,
    dense (1-byte) and sparse (5-byte) ones interleaved."""
    import torch

    cuda = torch.device("cuda", 0)
    rng = np.random.default_rng(13)
    parts, counts = [], []
    for l in range(400):
        target = int(rng.choice([511, 512, 513, 1023, 1024, 1025, 2047, 2048, 2049, 3000]))
        length = 1 if l % 2 else 5
        n = max(1, target // length)
        v = _values_of_lengths(rng, np.full(n, length))
        parts.append(oracle.encode_sequence(v))
        counts.append(n)
    byte_off = np.zeros(len(parts) + 1, np.uint64)
    byte_off[1:] = np.cumsum([p.size for p in parts])
    int_off = np.zeros(len(parts) + 1, np.uint64)
    int_off[1:] = np.cumsum(counts)
    data = np.concatenate(parts)
    prev = rng.integers(0, 1 << 32, len(parts), dtype=np.uint64).astype(np.uint32)
    out = torch.full((int(int_off[-1]) + 4,), -1, dtype=torch.int32, device=cuda)
    res = torch.zeros(len(parts) * 3, dtype=torch.int64, device=cuda)
    d = mvb.Decoder(cuda, 1 << 16)
    d.decode_lists(torch.from_numpy(data).to(cuda), torch.from_numpy(byte_off.view(np.int64)).to(cuda),
                   torch.from_numpy(int_off.view(np.int64)).to(cuda), out,
                   prev=torch.from_numpy(prev.view(np.int32)).to(cuda) if delta else None, results=res,
                   delta=delta)
    got = out.cpu().numpy().view(np.uint32)
    rr = res.cpu().numpy().reshape(-1, 3)
    for l, span in enumerate(parts):
        ro, oo = oracle.decode_delta(span, counts[l], int(prev[l])) if delta else oracle.decode(span, counts[l])
        assert tuple(int(x) for x in rr[l]) == tuple(ro), l
        assert np.array_equal(got[int(int_off[l]):int(int_off[l + 1])], oo), l


def _stream_with_long_ints_at(oracle, rng, base_lens, byte_positions, long_len):
    """Mostly 1-2-byte integers with one long_len-byte integer ending at (or
    just after) each requested byte position: the 1-2-byte slot path (prmt
    candidates, its lane / slice vote) next to slices that must not take it,
    and kernel A's 3+-byte detection (per-iteration sums plus the halo pair)."""
    lens = list(base_lens)
    pos = np.cumsum(lens)
    for bp in sorted(byte_positions, reverse=True):
        k = int(np.searchsorted(pos, bp))
        if k < len(lens):
            lens[k] = long_len
    lens = np.asarray(lens)
    return _values_of_lengths(rng, lens)


@pytest.mark.parametrize("long_len", [3, 4, 5])
def test_long_integers_at_lane_and_slice_seams(oracle, long_len):
    rng = np.random.default_rng(100 + long_len)
    base = rng.integers(1, 3, 60000)  # 1- and 2-byte integers (~90 KB)
    # around 32-byte lane seams, 512-byte and 1 KiB slice seams, segment seams
    seams = [32 * k + d for k in (3, 17, 31, 32, 33, 63) for d in (-2, -1, 0, 1, 2)]
    seams += [1024 * k + d for k in (1, 2, 7, 8, 40) for d in range(-4, 5)]
    seams += [512 * k + d for k in (3, 5) for d in (-1, 0, 1)]
    v = _stream_with_long_ints_at(oracle, rng, base, seams, long_len)
    enc = oracle.encode_sequence(v)
    r, out = gpu_decode(enc, v.size)
    assert r == (0, v.size, enc.size)
    assert np.array_equal(out, v)
    ro, oo = oracle.decode_delta(enc, v.size, 77)
    rd, od = gpu_decode(enc, v.size, delta=True, prev=77)
    assert rd == ro and np.array_equal(od, oo)
    # the same through the device path at a misaligned input and output
    rd2, od2 = dev_decode(__import__("torch"), __import__("torch").device("cuda", 0), enc, v.size, delta=True,
                          prev=77, in_off=5, out_off=3)
    assert rd2 == ro and np.array_equal(od2, oo)


def test_two_byte_slices_dense_and_sparse_mix(oracle):
    """Slices of only 1-byte integers (swizzled staging) and of only 2-byte
    integers, alternating every few KiB, plus single 3-byte integers between
    them: each slice decides its own path."""
    rng = np.random.default_rng(808)
    parts = []
    for i in range(60):
        n = int(rng.integers(500, 5000))
        parts.append(np.ones(n, np.int64) if i % 3 == 0 else np.full(n, 2, np.int64) if i % 3 == 1
                     else rng.integers(1, 3, n))
        if i % 7 == 3:
            parts.append(np.array([3], np.int64))
    v = _values_of_lengths(rng, np.concatenate(parts))
    enc = oracle.encode_sequence(v)
    r, out = gpu_decode(enc, v.size)
    assert r == (0, v.size, enc.size) and np.array_equal(out, v)
    ro, oo = oracle.decode_delta(enc, v.size, 5)
    rd, od = gpu_decode(enc, v.size, delta=True, prev=5)
    assert rd == ro and np.array_equal(od, oo)


def _mixed5(rng, n):
    """c1-like data: lengths uniform in 1..5, so nearly every slice holds
    5-byte integers (the plain fast path's 5-byte slots)."""
    return _values_of_lengths(rng, rng.integers(1, 6, n))


@pytest.mark.parametrize("delta", [False, True])
def test_mixed_five_byte_fifth_byte_checks(oracle, delta):
    """Strict mode's fifth-byte rule inside otherwise canonical 1..5-byte
    data: a 5-byte integer's fifth byte rewritten to 0x0F (largest valid),
    0x10, 0x7F (malformed: the slice must leave the fast path) or a
    continuation byte (a 6+-byte run), at lane / slice seams and mid-slice."""
    rng = np.random.default_rng(515)
    v = _mixed5(rng, 120_000)
    enc = oracle.encode_sequence(v)
    lens = 1 + sum((v >= (1 << s)).astype(np.int64) for s in (7, 14, 21, 28))
    ends = np.cumsum(lens) - 1
    fifth = ends[v >= (1 << 28)]  # byte index of each 5-byte integer's fifth byte
    picks = []
    for target in (31, 32, 33, 1023, 1024, 1025, 4096, 33_333, 70_001):
        picks.append(int(fifth[np.searchsorted(fifth, target)]))
    for pos in picks:
        for val in (0x0F, 0x10, 0x7F, 0x80):
            bad = enc.copy()
            bad[pos] = val
            if delta:
                ro, oo = oracle.decode_delta(bad, v.size, 3)
                r, out = gpu_decode(bad, v.size, delta=True, prev=3)
            else:
                ro, oo = oracle.decode(bad, v.size)
                r, out = gpu_decode(bad, v.size)
            assert r == ro and np.array_equal(out[: ro[1]], oo[: ro[1]]), (pos, val, delta)


@pytest.mark.parametrize("n", [1, 5, 31, 33, 257, 1000, 4097, 100_003])
def test_mixed_five_byte_ragged_sizes(oracle, n):
    """1..5-byte data at ragged sizes through the device path (misaligned
    input and output, guard words): tail slices of the plain fast path."""
    import torch

    rng = np.random.default_rng(9000 + n)
    v = _mixed5(rng, n)
    enc = oracle.encode_sequence(v)
    for delta in (False, True):
        ro, oo = oracle.decode_delta(enc, n, 17) if delta else oracle.decode(enc, n)
        r, out = dev_decode(torch, torch.device("cuda", 0), enc, n, STRICT, delta, 17, 3, 1)
        assert r == ro and np.array_equal(out, oo), (n, delta)
        # and one integer short of the stream (count-1 in the last slice)
        if n > 1:
            ro, oo = oracle.decode_delta(enc, n - 1, 17) if delta else oracle.decode(enc, n - 1)
            r, out = dev_decode(torch, torch.device("cuda", 0), enc, n - 1, STRICT, delta, 17, 0, 0)
            assert r == ro and np.array_equal(out, oo), (n, delta)


@pytest.mark.parametrize("delta", [False, True])
def test_lists_head_slices_on_two_byte_path(oracle, delta):
    """Lists of 1-2-byte integers starting at every offset inside a slice
    (the head slice's bytes before the list read as zeros and must store
    nothing), some count-limited inside the head slice, some with a 3-byte or
    malformed integer in it (those heads leave the 2-byte path)."""
    import torch

    cuda = torch.device("cuda", 0)
    rng = np.random.default_rng(4242)
    parts, counts, reqs = [], [], []
    for l in range(300):
        n = int(rng.integers(1, 900))
        lens = rng.integers(1, 3, n)
        if l % 11 == 5:
            lens[min(n - 1, int(rng.integers(0, 40)))] = 3
        enc = oracle.encode_sequence(_values_of_lengths(rng, lens))
        if l % 13 == 7 and enc.size > 12:
            enc = enc.copy()
            at = int(rng.integers(0, min(enc.size - 6, 60)))
            enc[at:at + 6] = 0x80
        gap = int(rng.integers(0, 64))  # junk bytes between lists: every start offset mod 16 / 512
        parts.append(rng.integers(0, 256, gap).astype(np.uint8))
        parts.append(enc)
        counts.append(n)
        reqs.append(n if l % 5 else max(1, int(rng.integers(1, min(n, 30) + 1))))
    sizes = [p.size for p in parts]
    starts = np.cumsum([0] + sizes)[1::2]  # byte offset of each list (after its junk gap)
    data = np.concatenate(parts)
    enc_sizes = np.array(sizes[1::2], np.int64)
    # the batch alternates list l (entry 2l) and the junk gap after it (entry 2l+1,
    # decoded too, ignored): byte_off[j] .. byte_off[j + 1] is entry j's bytes
    byte_off = np.concatenate([[s, s + z] for s, z in zip(starts, enc_sizes)]).astype(np.uint64)
    int_off = np.zeros(2 * len(counts), np.uint64)
    acc = 0
    for l, r in enumerate(reqs):
        int_off[2 * l] = acc
        int_off[2 * l + 1] = acc + r
        acc += r + 3  # a gap in the output between lists
    out = torch.full((acc + 4,), -1, dtype=torch.int32, device=cuda)
    n_b = 2 * len(counts) - 1  # lists 2l are ours; odd entries decode the junk gaps, ignored
    res = torch.zeros(n_b * 3, dtype=torch.int64, device=cuda)
    prev = rng.integers(0, 1 << 32, n_b, dtype=np.uint64).astype(np.uint32)
    d = mvb.Decoder(cuda, 1 << 16)
    d.decode_lists(torch.from_numpy(data).to(cuda), torch.from_numpy(byte_off.view(np.int64)).to(cuda),
                   torch.from_numpy(int_off.view(np.int64)).to(cuda), out,
                   prev=torch.from_numpy(prev.view(np.int32)).to(cuda) if delta else None, results=res, delta=delta)
    got = out.cpu().numpy().view(np.uint32)
    rr = res.cpu().numpy().reshape(-1, 3)
    for l in range(len(counts)):
        span = data[int(byte_off[2 * l]):int(byte_off[2 * l + 1])]
        r = reqs[l]
        ro, oo = oracle.decode_delta(span, r, int(prev[2 * l])) if delta else oracle.decode(span, r)
        assert tuple(int(x) for x in rr[2 * l]) == tuple(ro), l
        n = ro[1]
        assert np.array_equal(got[int(int_off[2 * l]):int(int_off[2 * l]) + n], oo[:n]), l
