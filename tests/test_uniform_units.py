"""Streams of equally long 4- and 5-byte integers (the per-integer gather of
decode_fused.cuh, unit_uniform) and everything that must make a unit fall
back: one integer of another length, a fifth byte >= 0x10, an over-long run,
a count limit, truncation -- plain and delta, at input misalignments, against
the oracle (decode_scalar / decode_delta_scalar, vbyte.cpp:47-74)."""
import numpy as np
import pytest

from oracle import STRICT
from test_decode_gpu import dev_decode

pytestmark = pytest.mark.gpu


def uniform_values(rng, n, length):
    lo = 1 << (7 * (length - 1))
    hi = min(1 << (7 * length), 1 << 32)
    return rng.integers(lo, hi, n, dtype=np.uint64).astype(np.uint32)


@pytest.mark.parametrize("delta", [False, True])
@pytest.mark.parametrize("length", [4, 5])
def test_uniform_streams_and_fallbacks(cuda, oracle, delta, length):
    import torch

    rng = np.random.default_rng(40 + length + 10 * delta)
    n = 60000  # ~60 units of 4 KiB
    v = uniform_values(rng, n, length)
    clean = oracle.encode_sequence(v)
    cases = [("clean", clean, n)]
    # a shorter / longer integer inside (that unit and the ones after it lose the shape or shift phase)
    for other in (1, 2, 3, 9 - length):
        w = v.copy()
        for pos in (7, 5000, 31000):
            w[pos] = uniform_values(rng, 1, other)[0]
        cases.append((f"other{other}", oracle.encode_sequence(w), n))
    e = clean.copy()
    if length == 5:
        e[5 * 20000 + 4] = 0x10 + 0x25  # a fifth byte >= 0x10: malformed at integer 20000
        cases.append(("fifth", e, n))
    e = clean.copy()
    e[length * 30000: length * 30000 + 7] = 0x80  # an over-long run
    cases.append(("run", e, n))
    cases.append(("count", clean, n - 12345))         # count limit inside a unit
    cases.append(("truncated", clean[:-2], n))        # the last integer unfinished
    for name, data, count in cases:
        for in_off in (0, 5):
            want_r, want = (oracle.decode_delta(data, count, 77) if delta else oracle.decode(data, count))
            got_r, got = dev_decode(torch, cuda, data, count, STRICT, delta=delta, prev=77, in_off=in_off, out_off=1)
            assert got_r == tuple(want_r), (name, in_off, got_r, want_r)
            k = want_r[1]
            np.testing.assert_array_equal(got[:k], want[:k], err_msg=f"{name} in_off={in_off}")


@pytest.mark.parametrize("delta", [False, True])
def test_uniform_phase_and_sizes(cuda, oracle, delta):
    """All-5-byte streams of sizes around unit multiples (every phase of the
    progression at a unit start), preceded by 0..4 one-byte integers."""
    import torch

    rng = np.random.default_rng(8)
    for lead in range(5):
        for n in (819, 820, 1638, 1639, 4096, 8191):
            v = np.concatenate([rng.integers(0, 128, lead, dtype=np.uint64).astype(np.uint32), uniform_values(rng, n, 5)])
            data = oracle.encode_sequence(v)
            want_r, want = (oracle.decode_delta(data, v.size, 3) if delta else oracle.decode(data, v.size))
            got_r, got = dev_decode(torch, cuda, data, v.size, STRICT, delta=delta, prev=3)
            assert got_r == tuple(want_r), (lead, n)
            np.testing.assert_array_equal(got, want, err_msg=f"lead={lead} n={n}")
