"""Pipelined host drop-in (mvb_decode_stream / mvb_decode_delta_stream on
strict streams of >= 4 MB by default): chunked H2D, one kernel pair per
chunk, D2H of each chunk's output range.  Forced onto small streams with
1-group (32 KiB) chunks here, so every chunk seam, the per-chunk integer
totals and the final DecodeResult are checked against the oracle, bit-exact."""
import numpy as np
import pytest

from oracle import STRICT
from paper_1503_07387_b200 import _lib, mvb
from paper_1503_07387_b200 import workload as W

pytestmark = pytest.mark.gpu


@pytest.fixture
def small_chunks():
    _lib.set_host_pipeline(0, 1, grow=False)  # every strict host decode pipelines, chunks of one group
    yield
    _lib.set_host_pipeline()


def host_decode(data, count, delta=False, prev=0):
    out = np.zeros(max(count, 1), np.uint32)
    if delta:
        r = mvb.decode_delta_stream(np.asarray(data, np.uint8), count, prev, out, mvb.DecodeOptions(mode=STRICT))
    else:
        r = mvb.decode_stream(np.asarray(data, np.uint8), count, out, mvb.DecodeOptions(mode=STRICT))
    return (int(r.status), r.values_written, r.bytes_consumed), out[:count]


def test_pipelined_sizes(oracle, small_chunks):
    for n in (1, 97, 4097, 30000, 100000, 300001):
        v = W.mixed_values(n, n + 3)
        enc = oracle.encode_sequence(v)
        r, out = host_decode(enc, n)
        assert r == (0, n, enc.size), n
        assert np.array_equal(out, v), n
        ro, oo = oracle.decode_delta(enc, n, 12345)
        rd, od = host_decode(enc, n, delta=True, prev=12345)
        assert rd == ro and np.array_equal(od, oo), n


def test_pipelined_dense_and_sparse(oracle, small_chunks):
    rng = np.random.default_rng(8)
    for v in (rng.integers(0, 128, 400000, dtype=np.uint64).astype(np.uint32),
              rng.integers(1 << 28, 2**32, 60000, dtype=np.uint64).astype(np.uint32)):
        enc = oracle.encode_sequence(v)
        r, out = host_decode(enc, v.size)
        assert r == (0, v.size, enc.size) and np.array_equal(out, v)
        ro, oo = oracle.decode_delta(enc, v.size, 1)
        rd, od = host_decode(enc, v.size, delta=True, prev=1)
        assert rd == ro and np.array_equal(od, oo)


def test_pipelined_count_stop_and_truncation(oracle, small_chunks):
    v = W.mixed_values(200000, 17)
    enc = oracle.encode_sequence(v)
    for count in (1, 5000, 77777, 199999, 200000, 250000):
        for delta in (False, True):
            ro, oo = oracle.decode_delta(enc, count, 3) if delta else oracle.decode(enc, count)
            r, out = host_decode(enc, count, delta, 3)
            assert r == ro, (count, delta)
            assert np.array_equal(out[: ro[1]], oo[: ro[1]]), (count, delta)
    for cut in (1, 32767, 32768, 32769, 100001, enc.size - 1):
        data = enc[:cut]
        ro, oo = oracle.decode(data, v.size)
        r, out = host_decode(data, v.size)
        assert r == ro and np.array_equal(out[: ro[1]], oo[: ro[1]]), cut


def test_pipelined_malformed_across_chunks(oracle, small_chunks):
    v = W.mixed_values(150000, 29)
    enc = oracle.encode_sequence(v)
    rng = np.random.default_rng(31)
    positions = [int(p) for p in rng.integers(0, enc.size - 64, 12)] + [32766, 32767, 65534, 98300]
    for pos in positions:
        for pat in ([0x80, 0x80, 0x80, 0x80, 0x80, 0x01], [0x81, 0x82, 0x83, 0x84, 0x20], [0x80] * 40):
            data = enc.copy()
            data[pos:pos + len(pat)] = pat
            for delta in (False, True):
                ro, oo = oracle.decode_delta(data, v.size, 9) if delta else oracle.decode(data, v.size)
                r, out = host_decode(data, v.size, delta, 9)
                assert r == ro, (pos, pat, delta)
                assert np.array_equal(out[: ro[1]], oo[: ro[1]]), (pos, pat, delta)


def test_pipelined_growing_chunks(oracle):
    """Doubling chunk sizes from one group: seams at 1, 3, 7, 15, ... groups."""
    _lib.set_host_pipeline(0, 1, grow=True)
    try:
        v = W.mixed_values(700000, 41)
        enc = oracle.encode_sequence(v)
        r, out = host_decode(enc, v.size)
        assert r == (0, v.size, enc.size) and np.array_equal(out, v)
        ro, oo = oracle.decode_delta(enc, v.size, 2)
        rd, od = host_decode(enc, v.size, delta=True, prev=2)
        assert rd == ro and np.array_equal(od, oo)
    finally:
        _lib.set_host_pipeline()


def test_pipelined_default_threshold_full_config2():
    """BASELINE config 2 at full size through the default (4 MB threshold,
    1 MB first chunk, doubling) pipelined drop-in, twice (the per-thread
    context is reused)."""
    w = W.config2()
    exp = w.expected()
    for _ in range(2):
        r, out = host_decode(w.encoded, w.count, delta=True, prev=w.prev)
        assert r == (0, w.count, w.encoded.size)
        assert np.array_equal(out, exp)


def _lists_batch(oracle, seed, n_lists=400):
    """Lists as in test_batched_lists_equal_per_list_oracle: empty ones,
    count-limited, truncated and malformed ones, an unaligned first start."""
    rng = np.random.default_rng(seed)
    parts, counts, prevs = [], [], []
    for l in range(n_lists):
        n = int(rng.integers(0, 3000)) if l % 7 else int(rng.integers(0, 4))
        v = W.mixed_values(n, l + 11) if n else np.zeros(0, np.uint32)
        e = oracle.encode_sequence(v) if n else np.zeros(0, np.uint8)
        cnt = n
        if l % 11 == 3 and n > 2:
            cnt = n - 2
        if l % 13 == 5 and e.size > 3:
            e = e[:-1]
        if l % 17 == 9 and e.size > 40:
            e = e.copy()
            e[20:26] = 0x80
        parts.append(e)
        counts.append(cnt)
        prevs.append(int(rng.integers(0, 1 << 32)))
    byte_off = np.zeros(n_lists + 1, np.uint64)
    byte_off[1:] = np.cumsum([p.size for p in parts])
    int_off = np.zeros(n_lists + 1, np.uint64)
    int_off[1:] = np.cumsum(counts)
    data = np.concatenate([np.zeros(5, np.uint8)] + parts)
    byte_off += 5
    return data, byte_off, int_off, parts, counts, np.array(prevs, np.uint32)


@pytest.mark.parametrize("delta", [True, False])
@pytest.mark.parametrize("grow", [False, True])
def test_host_lists_equal_per_list_oracle(oracle, delta, grow):
    """mvb_decode[_delta]_lists (host pointers, sub-batches pipelined; with
    1-byte sub-batch targets every list up to the 63rd is its own sub-batch)
    against one oracle decode per list."""
    data, byte_off, int_off, parts, counts, prevs = _lists_batch(oracle, 5 if delta else 6)
    _lib.set_host_pipeline(0, 1, grow=grow)
    try:
        out = np.full(int(int_off[-1]) + 4, 0xFFFFFFFF, np.uint32)
        res = mvb.decode_lists(data, byte_off, int_off, out, prev=prevs if delta else None, delta=delta)
    finally:
        _lib.set_host_pipeline()
    for l in range(len(parts)):
        span = data[int(byte_off[l]):int(byte_off[l + 1])]
        ro, oo = oracle.decode_delta(span, counts[l], int(prevs[l])) if delta else oracle.decode(span, counts[l])
        assert tuple(int(x) for x in res[l]) == tuple(ro), (l, res[l], ro)
        k = ro[1]
        np.testing.assert_array_equal(out[int(int_off[l]):int(int_off[l]) + k], oo[:k], err_msg=f"list {l}")
    assert out[int(int_off[-1]):].tolist() == [0xFFFFFFFF] * 4


def test_host_lists_config3_checksum():
    """BASELINE config 3 through the host batched entry (default sub-batches)."""
    w = W.config3()
    out = np.zeros(w.count, np.uint32)
    res = mvb.decode_lists(w.encoded, w.byte_offsets, w.int_offsets, out, delta=True)
    assert (res[:, 0] == 0).all()
    assert np.array_equal(out, w.expected())
