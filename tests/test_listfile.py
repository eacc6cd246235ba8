"""ListFile ingestion against the reference's own
reader/writer (core/src/list_file.cpp, through oracle/_ref), and the batched
GPU decode of ingested lists against one oracle decode per list."""
import io
import os

import numpy as np
import pytest

from oracle import Oracle, RefLib
from paper_1503_07387_b200 import listfile as LF
from paper_1503_07387_b200 import mvb
from paper_1503_07387_b200 import workload as W

ref_needed = pytest.mark.skipif(not RefLib.available(), reason="reference library not built")


def _lists(seed, n_lists=12):
    rng = np.random.default_rng(seed)
    out = []
    for l in range(n_lists):
        n = int(rng.integers(0, 2000))
        ids = np.unique(rng.integers(0, 1 << 25, n, dtype=np.int64)).astype(np.uint32)
        out.append(ids)
    return out


@ref_needed
def test_writer_and_reader_match_reference(tmp_path):
    ref = RefLib()
    for k, ids in enumerate(_lists(1)):
        buf = mvb.encode_deltas(ids)
        ours = tmp_path / f"o{k}.mvb"
        theirs = tmp_path / f"r{k}.mvb"
        LF.write_list_file(ours, buf, delta_coded=True)
        assert ref.write_list_file(theirs, buf.bytes, buf.count, True) == 0
        assert ours.read_bytes() == theirs.read_bytes()
        got = ref.read_list_file(ours)
        assert got is not None and np.array_equal(got[0], buf.bytes) and got[1] == buf.count and got[2]
        rec = LF.read_list_file(theirs)
        assert np.array_equal(rec.buf.bytes, buf.bytes) and rec.buf.count == buf.count and rec.delta_coded


@ref_needed
def test_default_flag_is_the_buffers_own(tmp_path):
    """write_list without an explicit flag writes buf.delta_coded
    (list_file.cpp:50), and read_list hands it back on the EncodedBuffer."""
    ref = RefLib()
    ids = np.array([3, 9, 200, 70000, 70001], np.uint32)
    for buf, want in ((mvb.encode_sequence(ids), False), (mvb.encode_deltas(ids), True)):
        path = tmp_path / f"d{int(want)}.mvb"
        LF.write_list_file(path, buf)
        got = ref.read_list_file(path)
        assert got is not None and got[2] == want
        rec = LF.read_list_file(path)
        assert rec.delta_coded == want and rec.buf.delta_coded == want
        again = tmp_path / f"a{int(want)}.mvb"
        LF.write_list_file(again, rec.buf)
        assert again.read_bytes() == path.read_bytes()


def _corruptions():
    good = mvb.encode_sequence(np.array([1, 300, 70000, 1 << 22, 0xFFFFFFFF], np.uint32))
    b = np.asarray(good.bytes, np.uint8)
    yield "ok", b, 5
    yield "count too high", b, 6
    yield "count too low", b, 4
    yield "extra byte", np.concatenate([b, [0x05]]), 5
    yield "truncated last", b[:-1], 5
    yield "six-byte int", np.array([0x81, 0x82, 0x83, 0x84, 0x85, 0x01], np.uint8), 1
    yield "fifth byte 0x10", np.array([0x81, 0x82, 0x83, 0x84, 0x10], np.uint8), 1
    yield "fifth byte 0x0F", np.array([0x81, 0x82, 0x83, 0x84, 0x0F], np.uint8), 1
    yield "non-minimal", np.array([0x85, 0x00], np.uint8), 1
    yield "empty ok", np.zeros(0, np.uint8), 0
    yield "empty count 1", np.zeros(0, np.uint8), 1


@ref_needed
@pytest.mark.parametrize("case", list(range(11)))
def test_validation_matches_reference(tmp_path, case):
    ref = RefLib()
    name, payload, count = list(_corruptions())[case]
    path = tmp_path / "x.mvb"
    assert ref.write_list_file(path, payload, count, False) == 0
    theirs_ok = ref.read_list_file(path, validate=True) is not None
    try:
        LF.read_list_file(path, validate_payload=True)
        ours_ok = True
    except LF.ListFileError:
        ours_ok = False
    assert ours_ok == theirs_ok, name
    # without validation both accept it
    assert ref.read_list_file(path, validate=False) is not None
    LF.read_list_file(path, validate_payload=False)


def test_header_errors(tmp_path):
    buf = mvb.encode_sequence(np.arange(100, dtype=np.uint32))
    f = io.BytesIO()
    LF.write_list(f, buf, delta_coded=False)
    raw = f.getvalue()
    for bad, msg in ((b"MVB2" + raw[4:], "bad magic"), (raw[:10], "truncated header"), (raw[:-1], "truncated payload"),
                     (b"", "bad magic")):
        with pytest.raises(LF.ListFileError, match=msg):
            LF.read_list(io.BytesIO(bad))


def test_batch_reads_back_to_back_containers(tmp_path):
    lists = _lists(2, 9)
    p1, p2 = tmp_path / "a.mvb", tmp_path / "b.mvb"
    with open(p1, "wb") as f:
        for ids in lists[:5]:
            LF.write_list(f, mvb.encode_deltas(ids), delta_coded=True)
    with open(p2, "wb") as f:
        for ids in lists[5:]:
            LF.write_list(f, mvb.encode_sequence(ids), delta_coded=False)
    b = LF.read_batch([p1, p2])
    assert b.n_lists == 9 and b.delta.tolist() == [True] * 5 + [False] * 4
    assert int(b.int_offsets[-1]) == sum(x.size for x in lists)
    assert int(b.byte_offsets[-1]) == b.payload.size


@pytest.mark.gpu
def test_batch_decode_on_gpu_equals_per_list_oracle(tmp_path):
    oracle = Oracle()
    lists = _lists(3, 40)
    lists.append(W.mixed_values(70000, 5))  # one long plain list
    path = tmp_path / "batch.mvb"
    with open(path, "wb") as f:
        for k, ids in enumerate(lists):
            if k % 3 == 2:  # plain list
                LF.write_list(f, mvb.encode_sequence(ids), delta_coded=False)
            else:
                LF.write_list(f, mvb.encode_deltas(np.sort(ids)), delta_coded=True)
    b = LF.read_batch(path)
    values, results = LF.decode_batch(b, "cuda:0")
    for l in range(b.n_lists):
        span = b.payload[int(b.byte_offsets[l]):int(b.byte_offsets[l + 1])]
        cnt = int(b.int_offsets[l + 1] - b.int_offsets[l])
        ro, oo = oracle.decode_delta(span, cnt, 0) if b.delta[l] else oracle.decode(span, cnt)
        assert tuple(int(x) for x in results[l]) == tuple(ro), l
        assert np.array_equal(values[int(b.int_offsets[l]):int(b.int_offsets[l + 1])], oo), l
