"""Regenerates tests/golden/*.json from the REFERENCE library itself.

Run in the build container (needs oracle/_ref/libmvb_ref.so, compiled from
/root/reference/proj/core/src by oracle/Makefile):

    make -C oracle && python tests/golden/make_golden.py

kat.json        known-answer cases: input bytes, count/prev/mode, the
                reference's DecodeResult and outputs (decode_scalar and
                decode_stream agree on all of them except where noted).
                Sources: vbyte_test.cpp, decode_test.cpp, acceptance.cpp and
                SURVEY.md Appendix A probes.
checksums.json  FNV-1a checksums (runner.cpp:63-72) of the input bytes and
                the reference's decoded output for larger seeded streams,
                including every BASELINE.json config, so the GPU tests can pin
                parity at full size without shipping the data.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import Oracle, RefLib, STRICT, PERMISSIVE  # noqa: E402
from paper_1503_07387_b200 import workload as W  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def hexs(b) -> str:
    return bytes(np.asarray(b, np.uint8)).hex()


def main():
    ref = RefLib()
    orc = Oracle()
    cases = []

    def add(name, data, count, mode=STRICT, delta=False, prev=0, note=""):
        data = np.asarray(bytearray(data) if isinstance(data, (bytes, list)) else data, np.uint8)
        if delta:
            r, out = ref.decode_delta_scalar(data, count, prev, mode)
            rs, outs = ref.decode_delta_stream(data, count, prev, mode)
        else:
            r, out = ref.decode_scalar(data, count, mode)
            rs, outs = ref.decode_stream(data, count, mode)
        n = r[1]
        cases.append({
            "name": name, "bytes": hexs(data), "count": count, "mode": mode, "delta": delta, "prev": prev,
            "status": r[0], "values_written": r[1], "bytes_consumed": r[2],
            "out": [int(x) for x in out[:n]],
            "stream_result": list(rs),
            "stream_agrees": bool(rs == r and np.array_equal(outs[:n], out[:n])),
            "note": note,
        })

    # Table 1 (vbyte_test.cpp:36-50, acceptance.cpp:48-66): encode + decode each row
    for v in (1, 2, 4, 128, 256, 512, 16384, 32768, 0, 4294967295):
        add(f"table1_{v}", bytes(ref.encode_sequence([v])), 1, note="encode_one row")
    # Fig. 1 (vbyte_test.cpp:97-116, decode_test.cpp:100-111, :284-292)
    fig1 = bytes([0x80, 0x01, 0x82, 0x03, 0x10, 0x20])
    add("fig1_plain", fig1, 4)
    add("fig1_delta_prev0", fig1, 4, delta=True)
    add("fig1_delta_prev100", fig1, 4, delta=True, prev=100)
    # window examples (decode_test.cpp:113-126) as streams
    add("ramp_1_to_16", bytes(range(1, 17)), 16)
    add("big_then_7", bytes([0x80, 0x80, 0x80, 0x80, 0x01, 0x07]), 2)
    add("zero_byte", bytes([0x00]), 1)
    add("empty_count0", b"", 0)
    add("empty_count1", b"", 1, note="no input: truncated at 0")
    # truncation (vbyte_test.cpp:140-151)
    t = bytes(ref.encode_sequence([5, 300]))[:-1]
    add("truncated_5_300", t, 2)
    add("truncated_5_300_delta", t, 2, delta=True, prev=7)
    # strict vs permissive fifth byte (vbyte_test.cpp:153-171)
    wide = bytes([0xFF] * 5)
    add("wide_strict", wide, 1)
    add("wide_permissive", wide, 1, mode=PERMISSIVE)
    six = bytes([0x80, 0x80, 0x80, 0x80, 0x80, 0x01])
    add("sixwide_strict", six, 2)
    add("sixwide_permissive", six, 2, mode=PERMISSIVE)
    # over-long integer inside a window-sized stream (decode_test.cpp:241-263)
    b = bytearray([0x01] * 64)
    for i in range(20, 25):
        b[i] = 0x80
    add("overlong_strict", bytes(b), 40)
    add("overlong_permissive", bytes(b), 40, mode=PERMISSIVE)
    add("overlong_permissive_delta", bytes(b), 40, mode=PERMISSIVE, delta=True, prev=3)
    # probe A.2: 5th byte 0x20 (scalar strict malformed; stream paths wrap)
    b = bytearray([0x01] * 64)
    b[20:25] = bytes([0x81, 0x82, 0x83, 0x84, 0x20])
    add("fifth_0x20_strict", bytes(b), 40, note="decode_stream returns ok here; GPU follows decode_scalar")
    add("fifth_0x20_permissive", bytes(b), 40, mode=PERMISSIVE)
    b2 = bytearray(b)
    b2[21:26] = bytes([0x80] * 5)
    add("six_byte_int_strict", bytes(b2), 40, note="progress counters differ between scalar and stream")
    add("six_byte_int_permissive", bytes(b2), 40, mode=PERMISSIVE)
    # permissive runs of 4..12 continuation bytes (probe A.2b), also a long one
    for L in list(range(4, 13)) + [17, 40]:
        b = bytearray([0x05] * 16) + bytearray([0x80 | (i * 37 % 128) for i in range(L)]) + bytearray([0x07]) \
            + bytearray([0x01] * 16)
        n_ints = 16 + (L + 1 + 4) // 5 + 16
        add(f"run{L}_permissive", bytes(b), n_ints, mode=PERMISSIVE)
        add(f"run{L}_permissive_delta", bytes(b), n_ints, mode=PERMISSIVE, delta=True, prev=11)
        add(f"run{L}_strict", bytes(b), n_ints)
    # stream ending in a run of continuation bytes
    for L in (1, 4, 5, 6, 9, 10, 11):
        b = bytearray([0x03] * 8) + bytearray([0x80] * L)
        add(f"tail_run{L}_strict", bytes(b), 8 + 4)
        add(f"tail_run{L}_permissive", bytes(b), 8 + 4, mode=PERMISSIVE)
    # truncated 50-int stream (decode_test.cpp:265-276)
    vals = W.mixed_values(50, 33)
    enc = ref.encode_sequence(vals)
    add("truncated_half_50", enc[: enc.size // 2], 50)
    # count stop (decode_test.cpp:223-239)
    vals = W.mixed_values(500, 9)
    add("count_stop_100_of_500", ref.encode_sequence(vals), 100)
    # all-zero gaps hold prev (decode_test.cpp:294-300)
    add("zero_gaps_prev42", ref.encode_sequence(np.zeros(100, np.uint32)), 100, delta=True, prev=42)
    # sizes sweep (decode_test.cpp:198-221), small ones inline
    for n in (1, 2, 11, 12, 13, 47, 48, 95, 96, 97):
        add(f"mixed_n{n}", ref.encode_sequence(W.mixed_values(n, n)), n)

    # oracle restatement must agree with the reference on every KAT
    for c in cases:
        data = np.frombuffer(bytes.fromhex(c["bytes"]), np.uint8)
        if c["delta"]:
            r, out = orc.decode_delta(data, c["count"], c["prev"], c["mode"])
        else:
            r, out = orc.decode(data, c["count"], c["mode"])
        assert list(r) == [c["status"], c["values_written"], c["bytes_consumed"]], c["name"]
        assert [int(x) for x in out[: r[1]]] == c["out"], c["name"]

    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py (reference library oracle/_ref)",
                   "cases": cases}, f, indent=1)

    # ---------------------------------------------------------- checksums
    sums = []

    def ck(name, values, delta=False, prev=0, mode=STRICT, count=None, enc=None, extra=None):
        enc = ref.encode_sequence(values) if enc is None else enc
        count = values.size if count is None else count
        if delta:
            r, out = ref.decode_delta_scalar(enc, count, prev, mode)
        else:
            r, out = ref.decode_scalar(enc, count, mode)
        rec = {"name": name, "delta": delta, "prev": prev, "mode": mode, "count": int(count),
               "in_len": int(enc.size), "in_fnv": orc.fnv_bytes(enc), "out_fnv": orc.fnv_u32(out[: r[1]]),
               "status": r[0], "values_written": r[1], "bytes_consumed": r[2]}
        if extra:
            rec.update(extra)
        sums.append(rec)
        print(name, rec["in_len"], r, flush=True)

    for n in (1000, 100000):
        ck(f"mixed_n{n}", W.mixed_values(n, n))
    ck("acceptance_fuzz_1e6_seed424242", W.mixed_values(1000000, 424242))
    g = W.mixed_values(20000, 77)
    for prev in (0, 1, 0xFFFFFFF0):
        ck(f"delta_mixed77_prev{prev}", g, delta=True, prev=prev)
    # BASELINE.json configs (full size, generated by paper_1503_07387_b200.workload)
    w = W.config1(); ck("config1", w.values, extra={"gen": "config1()"})
    w = W.config2(); ck("config2", w.values, delta=True, extra={"gen": "config2()"})
    for pt in W.C5_POINTS:
        w = W.config5(pt)
        ck(f"config5_{pt}_plain", w.values, enc=w.encoded, extra={"gen": f"config5('{pt}')"})
        ck(f"config5_{pt}_delta", w.values, enc=w.encoded, delta=True, extra={"gen": f"config5('{pt}', True)"})
    if "--c4" in sys.argv:
        w = W.config4(); ck("config4", w.values, enc=w.encoded, delta=True, extra={"gen": "config4()"})
        del w
    sums += extra_streams(ref, orc)
    with open(os.path.join(HERE, "checksums.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py (reference library oracle/_ref)",
                   "fnv": "FNV-1a 64 over bytes / little-endian u32 (tools/bench/runner.cpp:63-72)",
                   "streams": sums}, f, indent=1)


def permissive_c1_bytes():
    """config1's bytes with every 997th five-byte integer's fifth byte given
    high bits (0x70: strict rejects it, permissive keeps its low 4 bits) and
    every 50021st integer start overwritten by a 7-byte continuation run plus
    a terminator (permissive splits it into 5-byte chunks)."""
    w = W.config1()
    b = w.encoded.copy()
    term = np.flatnonzero(b < 0x80)
    starts = np.concatenate([[0], term[:-1] + 1])
    lens = term - starts + 1
    five = term[lens == 5]
    b[five[::997]] |= 0x70
    for st in starts[1000::50021]:
        if st + 8 < b.size:
            b[st:st + 7] = 0x81 + np.arange(7, dtype=np.uint8)
            b[st + 7] = 0x05
    return b


def extra_streams(ref, orc):
    """Reference checksums of config3 (the batch: one decode_delta_stream per
    list, runner.cpp:28-61) and of a full-size permissive stream."""
    out = []
    w = W.config3()
    enc = np.ascontiguousarray(w.encoded)
    bo = np.ascontiguousarray(w.byte_offsets.astype(np.uint64))
    io = np.ascontiguousarray(w.int_offsets.astype(np.uint64))
    vals = np.empty(w.count + 16, np.uint32)
    bad = ref.decode_delta_lists(enc, bo, io, vals, 0, bo.size - 1)
    out.append({"name": "config3", "delta": True, "prev": 0, "mode": STRICT, "count": int(w.count),
                "lists": int(bo.size - 1), "in_len": int(enc.size), "in_fnv": orc.fnv_bytes(enc),
                "offsets_fnv": orc.fnv_bytes(np.concatenate([bo.view(np.uint8), io.view(np.uint8)])),
                "out_fnv": orc.fnv_u32(vals[: w.count]), "lists_not_ok": int(bad), "gen": "config3()"})
    print("config3", enc.size, bad, flush=True)
    b = permissive_c1_bytes()
    for mode, tag in ((PERMISSIVE, "permissive"), (STRICT, "strict")):
        r, o = ref.decode_scalar(b, b.size, mode)  # every integer there is (truncated at the end)
        out.append({"name": f"config1_mutated_{tag}", "delta": False, "prev": 0, "mode": mode, "count": int(b.size),
                    "in_len": int(b.size), "in_fnv": orc.fnv_bytes(b), "out_fnv": orc.fnv_u32(o[: r[1]]),
                    "status": r[0], "values_written": r[1], "bytes_consumed": r[2],
                    "gen": "permissive_c1_bytes() (tests/golden/make_golden.py)"})
        print(f"config1_mutated_{tag}", b.size, r, flush=True)
    return out


if __name__ == "__main__":
    if "--extra-only" in sys.argv:  # append the extra streams to the existing checksums
        path = os.path.join(HERE, "checksums.json")
        with open(path) as f:
            d = json.load(f)
        extra = extra_streams(RefLib(), Oracle())
        names = {e["name"] for e in extra}
        d["streams"] = [e for e in d["streams"] if e["name"] not in names] + extra
        with open(path, "w") as f:
            json.dump(d, f, indent=1)
    else:
        main()
