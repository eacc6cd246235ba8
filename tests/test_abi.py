"""C-ABI library checks that need no GPU: the library loads, exports every
symbol include/mvb_cuda.h declares, and its host-side encoder agrees with the
oracle.  Decode calls without a device must fail loudly (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1503_07387_b200 import _lib, mvb
from paper_1503_07387_b200 import workload as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "mvb_cuda.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mvb_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 12
    assert set(syms) == set(_lib.EXPORTS)
    for s in syms:
        assert hasattr(L, s), s
    assert "sm_100a" in mvb.version()


def test_workload_library_loads():
    assert _lib.workload_lib().mvbw_encode is not None


def test_header_result_layout():
    assert ctypes.sizeof(_lib.MvbResult) == 24


def test_host_encoder_matches_oracle(oracle):
    for v in (0, 1, 127, 128, 16383, 16384, 2097151, 2097152, 268435455, 268435456, 4294967295):
        assert mvb.encode_one(v) == oracle.encode_one(v)
        assert mvb.encoded_size(v) == oracle.encoded_size(v)
    vals = W.mixed_values(20000, 3)
    buf = mvb.encode_sequence(vals)
    assert buf.count == vals.size and not buf.delta_coded
    assert np.array_equal(buf.bytes, oracle.encode_sequence(vals))
    assert np.array_equal(W.encode(vals), buf.bytes)  # multi-threaded bench encoder


def test_encode_deltas_semantics(oracle):
    s = np.sort(W.mixed_values(5000, 17))
    buf = mvb.encode_deltas(s)
    assert buf.delta_coded and buf.count == s.size
    r, out = oracle.decode_delta(buf.bytes, s.size, 0)
    assert r[0] == 0 and np.array_equal(out, s)
    with pytest.raises(ValueError):
        mvb.encode_deltas([3, 2])  # vbyte.cpp:80-81 throws std::invalid_argument
    assert mvb.delta_encode([1, 2, 3]).tolist() == [1, 1, 1]
    assert mvb.delta_encode([5, 5, 5]).tolist() == [5, 0, 0]
    with pytest.raises(ValueError):
        mvb.delta_encode([3, 2])
    assert mvb.prefix_sum_scalar([128, 386, 16, 32]).tolist() == [128, 514, 530, 562]
    assert mvb.encode_sequence([]).bytes.size == 0


def test_workspace_bytes_monotone():
    L = _lib.lib()
    prev = 0
    for n in (0, 1, 4095, 4096, 4097, 1 << 20, 1 << 30):
        b = L.mvb_workspace_bytes(n)
        assert b >= prev and b >= 256 + 32
        prev = b


def test_device_api_rejects_bad_arguments_without_touching_gpu():
    L = _lib.lib()
    # null input with nonzero length, null output with nonzero count, bad mode
    assert L.mvb_decode_device(None, 10, 1, None, 0, None, None, 0, None) == -1
    buf = (ctypes.c_uint8 * 16)()
    out = (ctypes.c_uint32 * 4)()
    assert L.mvb_decode_device(buf, 16, 1, out, 7, None, None, 0, None) == -1
    assert L.mvb_decode_device(buf, 16, 1, out, 0, None, None, 0, None) == -2  # no workspace


def test_decode_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(mvb.MvbError):
        mvb.decode_stream(bytes([1, 2, 3]), 3, np.zeros(3, np.uint32))
