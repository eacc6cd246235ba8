"""Parity of the sm_100a decoder (through the C ABI) with the oracle and the
reference's golden vectors.  Integer work: every comparison is bit-exact,
including DecodeResult's status, values_written and bytes_consumed."""
import os

import numpy as np
import pytest

from oracle import Oracle, PERMISSIVE, STRICT
from paper_1503_07387_b200 import mvb
from paper_1503_07387_b200 import workload as W

pytestmark = pytest.mark.gpu


def gpu_decode(data, count, mode=STRICT, delta=False, prev=0):
    """Host drop-in path: mvb_decode_stream / mvb_decode_delta_stream."""
    out = np.zeros(max(count, 1), np.uint32)
    if delta:
        r = mvb.decode_delta_stream(np.asarray(data, np.uint8), count, prev, out, mvb.DecodeOptions(mode=mode))
    else:
        r = mvb.decode_stream(np.asarray(data, np.uint8), count, out, mvb.DecodeOptions(mode=mode))
    return (int(r.status), r.values_written, r.bytes_consumed), out[:count]


def dev_decode(torch, dev, data, count, mode=STRICT, delta=False, prev=0, in_off=0, out_off=0):
    """Device path at chosen input/output misalignments (bytes / u32 words)."""
    data = np.asarray(data, np.uint8)
    src = torch.zeros(data.size + in_off + 16, dtype=torch.uint8, device=dev)
    src[in_off:in_off + data.size] = torch.from_numpy(data).to(dev)
    dst = torch.full((count + out_off + 8,), -1, dtype=torch.int32, device=dev)
    d = mvb._decoder_for(src)
    inp = src[in_off:in_off + data.size]
    out = dst[out_off:out_off + count]
    if delta:
        d.decode_delta(inp, count, prev, out, mode, in_len=data.size)
    else:
        d.decode(inp, count, out, mode, in_len=data.size)
    r = d.result()
    full = dst.cpu().numpy().view(np.uint32)
    # guard words around the output must be untouched (never writes past out+count)
    assert (full[:out_off] == 0xFFFFFFFF).all()
    assert (full[out_off + count:] == 0xFFFFFFFF).all()
    return (int(r.status), r.values_written, r.bytes_consumed), full[out_off:out_off + count]


def check_case(c, got):
    r, out = got
    n = c["values_written"]
    assert r == (c["status"], n, c["bytes_consumed"]), c["name"]
    assert out[:n].tolist() == c["out"], c["name"]


def test_kats_host_path(golden):
    kat, _ = golden
    for c in kat:
        data = np.frombuffer(bytes.fromhex(c["bytes"]), np.uint8)
        check_case(c, gpu_decode(data, c["count"], c["mode"], c["delta"], c["prev"]))


def test_kats_device_path_misaligned(golden, cuda):
    import torch

    kat, _ = golden
    for i, c in enumerate(kat):
        data = np.frombuffer(bytes.fromhex(c["bytes"]), np.uint8)
        for in_off, out_off in ((0, 0), (i % 16, i % 4), (15, 3), (7, 1)):
            check_case(c, dev_decode(torch, cuda, data, c["count"], c["mode"], c["delta"], c["prev"],
                                     in_off, out_off))


def test_sizes_sweep_equal_oracle(oracle):
    # decode_test.cpp:198-221 plus tile-boundary sizes
    for n in (1, 2, 11, 12, 13, 47, 48, 95, 96, 97, 1000, 1365, 1366, 4095, 4096, 4097, 100000, 300001):
        v = W.mixed_values(n, n)
        enc = oracle.encode_sequence(v)
        r, out = gpu_decode(enc, n)
        assert r == (0, n, enc.size), n
        assert np.array_equal(out, v), n
        rd, outd = gpu_decode(enc, n, delta=True, prev=n * 7919)
        ro, oo = oracle.decode_delta(enc, n, n * 7919)
        assert rd == ro and np.array_equal(outd, oo), n


def test_acceptance_stream_fuzz_1e6(oracle, golden):
    _, sums = golden
    s = sums["acceptance_fuzz_1e6_seed424242"]
    v = W.mixed_values(1000000, 424242)
    enc = oracle.encode_sequence(v)
    r, out = gpu_decode(enc, v.size)
    assert r == (s["status"], s["values_written"], s["bytes_consumed"])
    assert oracle.fnv_u32(out) == s["out_fnv"]


def test_delta_prev_wraparound(oracle, golden):
    _, sums = golden
    g = W.mixed_values(20000, 77)
    enc = oracle.encode_sequence(g)
    for prev in (0, 1, 0xFFFFFFF0):
        s = sums[f"delta_mixed77_prev{prev}"]
        r, out = gpu_decode(enc, g.size, delta=True, prev=prev)
        assert r == (s["status"], s["values_written"], s["bytes_consumed"])
        assert oracle.fnv_u32(out) == s["out_fnv"]


def test_count_stop_with_many_following(oracle):
    v = W.mixed_values(300000, 9)
    enc = oracle.encode_sequence(v)
    for count in (1, 100, 4097, 123457, 299999):
        r, out = gpu_decode(enc, count)
        ro, oo = oracle.decode(enc, count)
        assert r == ro and np.array_equal(out, oo), count
        r, out = gpu_decode(enc, count, delta=True, prev=5)
        ro, oo = oracle.decode_delta(enc, count, 5)
        assert r == ro and np.array_equal(out, oo), count


def _inject(enc, pos, pattern):
    b = enc.copy()
    b[pos:pos + len(pattern)] = pattern
    return b


def test_errors_at_random_positions_match_oracle(oracle):
    """Malformed / truncated / permissive-run cases inside long streams,
    including across tile (4 KiB) boundaries."""
    rng = np.random.default_rng(1234)
    v = W.mixed_values(60000, 4)
    enc = oracle.encode_sequence(v)
    patterns = [
        [0x80, 0x80, 0x80, 0x80, 0x80, 0x01],        # 6-byte integer
        [0x81, 0x82, 0x83, 0x84, 0x20],              # fifth byte 0x20
        [0xFF, 0xFF, 0xFF, 0xFF, 0x7F],              # fifth byte 0x7F
        [0x80] * 13 + [0x05],                        # long run
        [0x80] * 40,                                 # very long run
        [0x81, 0x82, 0x83, 0x84, 0x0F],              # canonical-length max fifth byte
    ]
    positions = [int(p) for p in rng.integers(0, enc.size - 64, 30)] + [4094, 4095, 4096, 4097, 8190, 12285]
    for pos in positions:
        for pat in patterns:
            data = _inject(enc, pos, pat)
            count = v.size
            for mode in (STRICT, PERMISSIVE):
                ro, oo = oracle.decode(data, count, mode)
                r, out = gpu_decode(data, count, mode)
                assert r == ro, (pos, pat, mode)
                assert np.array_equal(out[: ro[1]], oo[: ro[1]]), (pos, pat, mode)
                ro, oo = oracle.decode_delta(data, count, 99, mode)
                r, out = gpu_decode(data, count, mode, delta=True, prev=99)
                assert r == ro, (pos, pat, mode, "delta")
                assert np.array_equal(out[: ro[1]], oo[: ro[1]]), (pos, pat, mode, "delta")
        # truncation at pos
        data = enc[:pos]
        ro, oo = oracle.decode(data, v.size)
        r, out = gpu_decode(data, v.size)
        assert r == ro and np.array_equal(out[: ro[1]], oo[: ro[1]]), ("trunc", pos)


def test_all_continuation_permissive_stream(oracle):
    for n in (4, 5, 9, 10, 4096, 4100, 20000):
        data = np.full(n, 0x80 | 0x35, np.uint8)
        data[::7] = 0xFF
        count = n // 5 + 2
        for mode in (STRICT, PERMISSIVE):
            ro, oo = oracle.decode(data, count, mode)
            r, out = gpu_decode(data, count, mode)
            assert r == ro and np.array_equal(out[: ro[1]], oo[: ro[1]]), (n, mode)


def test_window_structures_all_masks(oracle):
    """acceptance.cpp:192-243 replayed as 16-byte streams: every 12-bit
    continuation mask with random payloads, strict and permissive."""
    rng = np.random.default_rng(2024)
    windows = []
    for m in range(4096):
        for _ in range(2):
            w = rng.integers(0, 128, 16, dtype=np.uint8)
            for i in range(12):
                if (m >> i) & 1:
                    w[i] |= 0x80
            w[12:] = rng.integers(0, 128, 4, dtype=np.uint8)
            windows.append(w)
    # concatenating the windows gives one long adversarial stream too
    big = np.concatenate(windows)
    for mode in (STRICT, PERMISSIVE):
        count = big.size
        ro, oo = oracle.decode(big, count, mode)
        r, out = gpu_decode(big, count, mode)
        assert r == ro and np.array_equal(out[: ro[1]], oo[: ro[1]]), mode
    for w in windows[::37]:
        for mode in (STRICT, PERMISSIVE):
            ro, oo = oracle.decode(w, 12, mode)
            r, out = gpu_decode(w, 12, mode)
            assert r == ro and np.array_equal(out[: ro[1]], oo[: ro[1]])


def test_five_byte_integers_across_tile_boundaries(oracle):
    rng = np.random.default_rng(5)
    for lead in range(0, 8):
        v = np.concatenate([np.full(lead, 3, np.uint32),
                            rng.integers(1 << 28, 2**32, 3000, dtype=np.uint64).astype(np.uint32)])
        enc = oracle.encode_sequence(v)
        r, out = gpu_decode(enc, v.size)
        assert r == (0, v.size, enc.size) and np.array_equal(out, v)


def test_sorted_lists_round_trip():
    # acceptance.cpp:287-312 structure: lengths in [2^4, 2^16], sorted uniform ids
    rng = np.random.default_rng(777)
    for _ in range(60):
        e = int(rng.integers(4, 16))
        n = int(rng.integers(1 << e, min((1 << (e + 1)) - 1, 1 << 16) + 1))
        s = np.sort(rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32))
        buf = mvb.encode_deltas(s)
        got = np.zeros(n, np.uint32)
        r = mvb.decode_delta_stream(buf, 0, got)
        assert r.status == mvb.DecodeStatus.ok and np.array_equal(got, s)


def test_back_to_back_reuse_and_epochs(oracle, cuda):
    """Many launches on one workspace (epoch-tagged lookback), sizes shrinking
    and growing, interleaved with failing decodes."""
    import torch

    rng = np.random.default_rng(11)
    d = mvb.Decoder(cuda, capacity_bytes=1 << 22)
    for it in range(40):
        n = int(rng.integers(1, 200000))
        v = W.mixed_values(n, it)
        enc = oracle.encode_sequence(v)
        if it % 5 == 3:
            enc = enc[: enc.size // 2]
        src = torch.from_numpy(enc).to(cuda)
        out = torch.zeros(n, dtype=torch.int32, device=cuda)
        d.decode(src, n, out)
        r = d.result()
        ro, oo = oracle.decode(enc, n)
        assert (int(r.status), r.values_written, r.bytes_consumed) == ro
        assert np.array_equal(out.cpu().numpy().view(np.uint32)[: ro[1]], oo[: ro[1]])


def test_empty_and_zero_count():
    r, _ = gpu_decode(np.zeros(0, np.uint8), 0)
    assert r == (0, 0, 0)
    r, _ = gpu_decode(np.zeros(0, np.uint8), 3)
    assert r == (1, 0, 0)
    r, _ = gpu_decode(np.array([1, 2, 3], np.uint8), 0)
    assert r == (0, 0, 0)


@pytest.mark.parametrize("name", ["config1", "config2"] + [f"config5_{p}_{k}" for p in W.C5_POINTS
                                                            for k in ("plain", "delta")])
def test_full_size_configs_checksums(name, golden, oracle):
    _, sums = golden
    s = sums[name]
    if name == "config1":
        w = W.config1()
    elif name == "config2":
        w = W.config2()
    else:
        _, pt, kind = name.split("_")
        w = W.config5(pt, kind == "delta")
    assert oracle.fnv_bytes(w.encoded) == s["in_fnv"]
    r, out = gpu_decode(w.encoded, w.count, delta=s["delta"], prev=s["prev"])
    assert r == (s["status"], s["values_written"], s["bytes_consumed"])
    assert oracle.fnv_u32(out) == s["out_fnv"]
    assert np.array_equal(out, w.expected())


@pytest.mark.parametrize("tag", ["permissive", "strict"])
def test_full_size_permissive_stream(tag, golden, oracle):
    """A full-size (config1, 50 MB) stream with non-canonical fifth bytes and
    7-byte continuation runs: permissive mode splits and masks them exactly as
    the reference does (decode_test.cpp:241-263 at size), strict mode stops at
    the first one; pinned by the reference's own checksums."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("make_golden", os.path.join(os.path.dirname(__file__), "golden",
                                                                              "make_golden.py"))
    mg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mg)
    b = mg.permissive_c1_bytes()
    _, sums = golden
    s = sums[f"config1_mutated_{tag}"]
    assert oracle.fnv_bytes(b) == s["in_fnv"]
    r, out = gpu_decode(b, s["count"], s["mode"])
    assert r == (s["status"], s["values_written"], s["bytes_consumed"])
    assert oracle.fnv_u32(out[: r[1]]) == s["out_fnv"]


def test_config3_batch_matches_reference_checksum(golden, oracle, cuda):
    """The c3 batch (65,536 lists) in one batched launch against the
    reference's per-list decode_delta_stream output (checksum)."""
    import torch

    _, sums = golden
    s = sums["config3"]
    w = W.config3()
    assert oracle.fnv_bytes(w.encoded) == s["in_fnv"]
    bo = w.byte_offsets.astype(np.uint64)
    io = w.int_offsets.astype(np.uint64)
    out = torch.empty(w.count, dtype=torch.int32, device=cuda)
    res = torch.zeros(3 * (bo.size - 1), dtype=torch.int64, device=cuda)
    d = mvb.Decoder(cuda, 1 << 12)
    d.decode_lists(torch.from_numpy(w.encoded).to(cuda), torch.from_numpy(bo.view(np.int64)).to(cuda),
                   torch.from_numpy(io.view(np.int64)).to(cuda), out, results=res, delta=True)
    rr = res.cpu().numpy().reshape(-1, 3)
    assert int((rr[:, 0] != 0).sum()) == s["lists_not_ok"]
    assert oracle.fnv_u32(out.cpu().numpy().view(np.uint32)) == s["out_fnv"]


def test_config4_full_size_device(golden, oracle, cuda):
    import torch

    _, sums = golden
    s = sums["config4"]
    w = W.config4()
    assert w.encoded.size == s["in_len"]
    src = torch.from_numpy(w.encoded).to(cuda)
    out = torch.empty(w.count, dtype=torch.int32, device=cuda)
    d = mvb.Decoder(cuda)
    d.decode_delta(src, w.count, 0, out)
    r = d.result()
    assert (int(r.status), r.values_written, r.bytes_consumed) == (s["status"], s["values_written"],
                                                                  s["bytes_consumed"])
    got = out.cpu().numpy().view(np.uint32)
    assert oracle.fnv_u32(got) == s["out_fnv"]


@pytest.mark.parametrize("choice", [1, 6, 0])
def test_every_strict_kernel_variant(choice, golden, oracle):
    """All strict-mode kernels (per-tile, warp-tile, CTA-pipelined, warp-sliced) agree with
    the oracle on KATs, errors across tile boundaries and a full config."""
    from paper_1503_07387_b200 import _lib

    _lib.set_kernel_choice(choice)
    try:
        kat, sums = golden
        for c in kat:
            if c["mode"] != STRICT:
                continue
            data = np.frombuffer(bytes.fromhex(c["bytes"]), np.uint8)
            check_case(c, gpu_decode(data, c["count"], c["mode"], c["delta"], c["prev"]))
        v = W.mixed_values(70000, 8)
        enc = oracle.encode_sequence(v)
        for pos in (0, 511, 512, 513, 4095, 4096, 9000, 40001):
            data = _inject(enc, pos, [0x80] * 6)
            for count in (v.size, 5000):
                ro, oo = oracle.decode(data, count)
                r, out = gpu_decode(data, count)
                assert r == ro and np.array_equal(out[: ro[1]], oo[: ro[1]]), (choice, pos, count)
                ro, oo = oracle.decode_delta(data, count, 3)
                r, out = gpu_decode(data, count, delta=True, prev=3)
                assert r == ro and np.array_equal(out[: ro[1]], oo[: ro[1]]), (choice, pos, count)
        for n in (1, 3, 600, 100001):
            w = W.mixed_values(n, n + 1)
            e = oracle.encode_sequence(w)
            for cut in (e.size, max(1, e.size - 3)):
                ro, oo = oracle.decode(e[:cut], n)
                r, out = gpu_decode(e[:cut], n)
                assert r == ro and np.array_equal(out[: ro[1]], oo[: ro[1]]), (choice, n, cut)
        s = sums["config2"]
        w = W.config2()
        r, out = gpu_decode(w.encoded, w.count, delta=True)
        assert r == (s["status"], s["values_written"], s["bytes_consumed"])
        assert oracle.fnv_u32(out) == s["out_fnv"]
    finally:
        _lib.set_kernel_choice(0)


def test_workspace_reuse_across_sizes_modes_and_kernels(cuda, oracle):
    """One Decoder (one workspace) serving decodes of different sizes, both
    modes and every strict kernel: accumulators left by one launch layout must
    never leak into another (they live at size-dependent offsets)."""
    import torch

    from paper_1503_07387_b200 import _lib

    d = mvb.Decoder(cuda, 1 << 20)
    streams = []
    for n, seed in ((300000, 1), (700, 2), (60000, 3), (5, 4), (150000, 5)):
        v = W.mixed_values(n, seed)
        streams.append((v, oracle.encode_sequence(v)))
    try:
        for choice in (0, 1, 6, 0):
            _lib.set_kernel_choice(choice)
            for rep in range(2):
                for (v, enc), mode in zip(streams * 2, [STRICT] * 5 + [PERMISSIVE] * 5):
                    src = torch.from_numpy(enc).to(cuda)
                    out = torch.empty(v.size, dtype=torch.int32, device=cuda)
                    d.decode_delta(src, v.size, 9, out, mode)
                    r = d.result()
                    ro, oo = oracle.decode_delta(enc, v.size, 9, mode)
                    assert (int(r.status), r.values_written, r.bytes_consumed) == tuple(ro), (choice, v.size, mode)
                    assert np.array_equal(out.cpu().numpy().view(np.uint32), oo), (choice, v.size, mode)
    finally:
        _lib.set_kernel_choice(0)


@pytest.mark.parametrize("choice", [0, 6])
@pytest.mark.parametrize("delta", [True, False])
def test_batched_lists_equal_per_list_oracle(cuda, oracle, delta, choice):
    """mvb_decode[_delta]_lists_device against one oracle decode per list,
    including empty lists, count-limited lists (more bytes than integers),
    truncated and malformed lists, unaligned list starts and a longest-first
    order."""
    import torch

    rng = np.random.default_rng(77)
    parts, counts, prevs = [], [], []
    for l in range(700):
        n = int(rng.integers(0, 3000)) if l % 7 else int(rng.integers(0, 4))
        v = W.mixed_values(n, l + 1) if n else np.zeros(0, np.uint32)
        e = oracle.encode_sequence(v) if n else np.zeros(0, np.uint8)
        cnt = n
        if l % 11 == 3 and n > 2:
            cnt = n - 2  # span holds more integers than requested
        if l % 13 == 5 and e.size > 3:
            e = e[:-1]   # truncated last integer
        if l % 17 == 9 and e.size > 40:
            e = e.copy()
            e[20:26] = 0x80  # over-long run: malformed
        parts.append(e)
        counts.append(cnt)
        prevs.append(int(rng.integers(0, 1 << 32)))
    byte_off = np.zeros(len(parts) + 1, np.uint64)
    byte_off[1:] = np.cumsum([p.size for p in parts])
    int_off = np.zeros(len(parts) + 1, np.uint64)
    int_off[1:] = np.cumsum(counts)
    data = np.concatenate([np.zeros(3, np.uint8)] + parts)  # 3-byte offset: unaligned list starts
    byte_off += 3
    src = torch.from_numpy(data).to(cuda)
    out = torch.full((int(int_off[-1]) + 4,), -1, dtype=torch.int32, device=cuda)
    res = torch.zeros(len(parts) * 3, dtype=torch.int64, device=cuda)
    order = np.argsort(-np.diff(byte_off).astype(np.int64), kind="stable").astype(np.uint32)
    from paper_1503_07387_b200 import _lib

    d = mvb.Decoder(cuda, 1 << 16)
    _lib.set_kernel_choice(choice)
    try:
        d.decode_lists(src, torch.from_numpy(byte_off.view(np.int64)).to(cuda),
                       torch.from_numpy(int_off.view(np.int64)).to(cuda), out,
                       prev=torch.from_numpy(np.array(prevs, np.uint32).view(np.int32)).to(cuda) if delta else None,
                       order=torch.from_numpy(order.view(np.int32)).to(cuda), results=res, delta=delta)
    finally:
        _lib.set_kernel_choice(0)
    got = out.cpu().numpy().view(np.uint32)
    rr = res.cpu().numpy().reshape(-1, 3)
    for l, e in enumerate(parts):
        span = data[int(byte_off[l]):int(byte_off[l + 1])]
        if delta:
            ro, oo = oracle.decode_delta(span, counts[l], prevs[l])
        else:
            ro, oo = oracle.decode(span, counts[l])
        assert tuple(int(x) for x in rr[l]) == tuple(ro), (l, rr[l], ro)
        k = ro[1]
        np.testing.assert_array_equal(got[int(int_off[l]):int(int_off[l]) + k], oo[:k], err_msg=f"list {l}")
    assert got[int(int_off[-1]):].tolist() == [0xFFFFFFFF] * 4  # nothing past the last list's output


def test_device_encoder_matches_reference_encoder(cuda, oracle):
    """mvb_encode_sequence_device / mvb_encode_deltas_device byte-for-byte
    against the reference encoder, across sizes and tile edges; decreasing
    input reports the first bad index like encode_deltas throws."""
    import torch

    for n in (0, 1, 5, 4095, 4096, 4097, 100003, 1 << 20):
        v = W.mixed_values(n, n + 3) if n else np.zeros(0, np.uint32)
        got = mvb.encode_device(torch.from_numpy(v.view(np.int32)).to(cuda)).cpu().numpy()
        np.testing.assert_array_equal(got, oracle.encode_sequence(v), err_msg=f"n={n}")
        s = np.sort(v)
        got = mvb.encode_device(torch.from_numpy(s.view(np.int32)).to(cuda), deltas=True).cpu().numpy()
        gaps = np.diff(np.concatenate([[0], s.astype(np.int64)])).astype(np.uint32)
        np.testing.assert_array_equal(got, oracle.encode_sequence(gaps), err_msg=f"deltas n={n}")
    # input and output at odd alignments (the encoder's vector loads and aligned chunk stores)
    v = W.mixed_values(70001, 9)
    for off in (1, 2, 3):
        t = torch.zeros(v.size + 8, dtype=torch.int32, device=cuda)
        t[off:off + v.size] = torch.from_numpy(v.view(np.int32)).to(cuda)
        got = mvb.encode_device(t[off:off + v.size]).cpu().numpy()
        np.testing.assert_array_equal(got, oracle.encode_sequence(v), err_msg=f"input offset {off}")
    v = np.sort(W.mixed_values(50000, 1))
    v[31337] = v[31336] - 1 if v[31336] else 5
    v[40000] = 0
    with pytest.raises(ValueError, match="index 31337" if v[31336] else "index"):
        mvb.encode_device(torch.from_numpy(v.view(np.int32)).to(cuda), deltas=True)
    # round trip through the device decoder
    w = W.config2(1 << 20)
    enc = mvb.encode_device(torch.from_numpy(w.values.view(np.int32)).to(cuda))
    out = torch.empty(w.count, dtype=torch.int32, device=cuda)
    d = mvb.Decoder(cuda, enc.numel())
    d.decode_delta(enc, w.count, 0, out)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), w.expected())


@pytest.mark.parametrize("buffer_ints", [1, 7, 4096])
def test_chunked_l1_mode_equals_full(oracle, buffer_ints):
    """The reference runner's l1 buffer mode (chunks of buffer_ints through a
    reused buffer, bytes_consumed and prev carried across calls) through the
    GPU drop-in equals one full decode (runner.cpp:28-61)."""
    rng = np.random.default_rng(buffer_ints)
    for n in (1, 4095, 4096, 50001):
        ids = np.unique(rng.integers(0, 1 << 25, n, dtype=np.int64)).astype(np.uint32)
        buf = mvb.encode_deltas(ids)
        full = np.zeros(ids.size, np.uint32)
        l1 = np.zeros(ids.size, np.uint32)
        assert mvb.decode_list(buf, full, "full").status == mvb.DecodeStatus.ok
        r = mvb.decode_list(buf, l1, "l1", buffer_ints)
        assert r.status == mvb.DecodeStatus.ok
        np.testing.assert_array_equal(full, ids)
        np.testing.assert_array_equal(l1, ids)
