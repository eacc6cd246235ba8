"""TEST INFRASTRUCTURE ONLY -- ctypes wrappers for the CPU checkers.

  Oracle()     oracle/liboracle.so: plain-C restatement of the reference's
               scalar codec (mvb_oracle.c, each function cites its reference
               lines).  Pinned against RefLib and tests/golden/.
  RefLib()     oracle/_ref/libmvb_ref.so: the UNMODIFIED reference library
               compiled from /root/reference/proj/core/src (oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may use
this package; the product decode path never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmvb_ref.so")

STRICT, PERMISSIVE = 0, 1


class Result(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("values_written", ctypes.c_uint64), ("bytes_consumed", ctypes.c_uint64)]

    def tuple(self):
        return (int(self.status), int(self.values_written), int(self.bytes_consumed))


def build(ref: bool = True) -> None:
    """make -C oracle (liboracle.so; and _ref/ when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "all" if ref else os.path.join(HERE, "liboracle.so")],
                   check=True)


def _p(a: np.ndarray) -> Optional[int]:
    return a.ctypes.data if a.size else None


def _u8(b) -> np.ndarray:
    if isinstance(b, (bytes, bytearray)):
        return np.frombuffer(bytes(b), np.uint8)
    return np.ascontiguousarray(b, dtype=np.uint8)


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = ctypes.CDLL(path)
        vp, sz, u32, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_int
        L.oracle_encoded_size.argtypes = [u32]; L.oracle_encoded_size.restype = sz
        L.oracle_encode_one.argtypes = [u32, vp]; L.oracle_encode_one.restype = sz
        L.oracle_encode_sequence.argtypes = [vp, sz, vp]; L.oracle_encode_sequence.restype = sz
        L.oracle_encoded_length.argtypes = [vp, sz]; L.oracle_encoded_length.restype = sz
        L.oracle_decode.argtypes = [vp, sz, sz, vp, i32]; L.oracle_decode.restype = Result
        L.oracle_decode_delta.argtypes = [vp, sz, sz, u32, vp, i32]; L.oracle_decode_delta.restype = Result
        L.oracle_delta_encode.argtypes = [vp, sz, vp, ctypes.POINTER(sz)]; L.oracle_delta_encode.restype = i32
        L.oracle_prefix_sum.argtypes = [vp, sz, u32, vp]; L.oracle_prefix_sum.restype = None
        L.oracle_fnv1a_u32.argtypes = [vp, sz, ctypes.c_uint64]; L.oracle_fnv1a_u32.restype = ctypes.c_uint64
        L.oracle_fnv1a_bytes.argtypes = [vp, sz, ctypes.c_uint64]; L.oracle_fnv1a_bytes.restype = ctypes.c_uint64
        self.L = L

    def encoded_size(self, x: int) -> int:
        return int(self.L.oracle_encoded_size(x))

    def encode_one(self, x: int) -> bytes:
        b = (ctypes.c_uint8 * 5)()
        n = self.L.oracle_encode_one(x, b)
        return bytes(b[:n])

    def encode_sequence(self, values) -> np.ndarray:
        v = np.ascontiguousarray(values, dtype=np.uint32)
        out = np.empty(self.L.oracle_encoded_length(_p(v), v.size), np.uint8)
        self.L.oracle_encode_sequence(_p(v), v.size, _p(out))
        return out

    def decode(self, data, count: int, mode: int = STRICT):
        src = _u8(data)
        out = np.zeros(max(count, 0), np.uint32)
        r = self.L.oracle_decode(_p(src), src.size, count, _p(out), mode)
        return r.tuple(), out

    def decode_delta(self, data, count: int, prev: int, mode: int = STRICT):
        src = _u8(data)
        out = np.zeros(max(count, 0), np.uint32)
        r = self.L.oracle_decode_delta(_p(src), src.size, count, prev & 0xFFFFFFFF, _p(out), mode)
        return r.tuple(), out

    def prefix_sum(self, gaps, prev: int = 0) -> np.ndarray:
        g = np.ascontiguousarray(gaps, dtype=np.uint32)
        out = np.empty_like(g)
        self.L.oracle_prefix_sum(_p(g), g.size, prev & 0xFFFFFFFF, _p(out))
        return out

    def fnv_u32(self, a, h: int = 0xCBF29CE484222325) -> int:
        a = np.ascontiguousarray(a, dtype=np.uint32)
        return int(self.L.oracle_fnv1a_u32(_p(a), a.size, h))

    def fnv_bytes(self, a, h: int = 0xCBF29CE484222325) -> int:
        a = _u8(a)
        return int(self.L.oracle_fnv1a_bytes(_p(a), a.size, h))


class RefLib:
    """The reference library itself (built from /root/reference sources)."""

    AUTO, PORTABLE, VECTOR = 0, 1, 2

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = ctypes.CDLL(path)
        vp, sz, u32, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_int
        L.mvbref_vector_available.restype = i32
        L.mvbref_encode_sequence.argtypes = [vp, sz, vp]; L.mvbref_encode_sequence.restype = sz
        L.mvbref_encode_deltas.argtypes = [vp, sz, vp]; L.mvbref_encode_deltas.restype = sz
        L.mvbref_decode_scalar.argtypes = [vp, sz, sz, vp, i32]; L.mvbref_decode_scalar.restype = Result
        L.mvbref_decode_delta_scalar.argtypes = [vp, sz, sz, u32, vp, i32]
        L.mvbref_decode_delta_scalar.restype = Result
        L.mvbref_decode_stream.argtypes = [vp, sz, sz, vp, i32, i32, sz]; L.mvbref_decode_stream.restype = Result
        L.mvbref_decode_delta_stream.argtypes = [vp, sz, sz, u32, vp, i32, i32, sz]
        L.mvbref_decode_delta_stream.restype = Result
        L.mvbref_decode_delta_lists.argtypes = [vp, vp, vp, vp, sz, sz]
        L.mvbref_decode_delta_lists.restype = sz
        L.mvbref_write_list_file.argtypes = [ctypes.c_char_p, vp, sz, u32, i32]
        L.mvbref_write_list_file.restype = i32
        L.mvbref_read_list_file.argtypes = [ctypes.c_char_p, i32, vp, sz, ctypes.POINTER(u32), ctypes.POINTER(i32)]
        L.mvbref_read_list_file.restype = ctypes.c_longlong
        self.L = L

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def vector_available(self) -> bool:
        return bool(self.L.mvbref_vector_available())

    def encode_sequence(self, values) -> np.ndarray:
        v = np.ascontiguousarray(values, dtype=np.uint32)
        n = self.L.mvbref_encode_sequence(_p(v), v.size, None)
        out = np.empty(n, np.uint8)
        self.L.mvbref_encode_sequence(_p(v), v.size, _p(out))
        return out

    def encode_deltas(self, values):
        v = np.ascontiguousarray(values, dtype=np.uint32)
        n = self.L.mvbref_encode_deltas(_p(v), v.size, None)
        if n == ctypes.c_size_t(-1).value:
            raise ValueError("reference encode_deltas: input decreases")
        out = np.empty(n, np.uint8)
        self.L.mvbref_encode_deltas(_p(v), v.size, _p(out))
        return out

    def decode_scalar(self, data, count: int, mode: int = STRICT, out: Optional[np.ndarray] = None):
        src = _u8(data)
        out = np.zeros(max(count, 0), np.uint32) if out is None else out
        r = self.L.mvbref_decode_scalar(_p(src), src.size, count, _p(out), mode)
        return r.tuple(), out

    def decode_delta_scalar(self, data, count: int, prev: int, mode: int = STRICT,
                            out: Optional[np.ndarray] = None):
        src = _u8(data)
        out = np.zeros(max(count, 0), np.uint32) if out is None else out
        r = self.L.mvbref_decode_delta_scalar(_p(src), src.size, count, prev & 0xFFFFFFFF, _p(out), mode)
        return r.tuple(), out

    def decode_stream(self, data, count: int, mode: int = STRICT, path: int = 0, handoff: int = 0,
                      out: Optional[np.ndarray] = None):
        src = _u8(data)
        out = np.zeros(max(count, 0) + 4, np.uint32) if out is None else out
        r = self.L.mvbref_decode_stream(_p(src), src.size, count, _p(out), mode, path, handoff)
        return r.tuple(), out[:count]

    def write_list_file(self, path, payload, count: int, delta: bool) -> int:
        b = _u8(payload)
        return int(self.L.mvbref_write_list_file(str(path).encode(), _p(b), b.size, count, int(delta)))

    def read_list_file(self, path, validate: bool = True):
        """(payload, count, delta) or None on the reference's ListFileError."""
        cap = max(os.path.getsize(path), 1)
        out = np.zeros(cap, np.uint8)
        cnt, dl = ctypes.c_uint32(0), ctypes.c_int32(0)
        n = int(self.L.mvbref_read_list_file(str(path).encode(), int(validate), _p(out), cap, ctypes.byref(cnt),
                                             ctypes.byref(dl)))
        if n < 0:
            return None
        return out[:n], int(cnt.value), bool(dl.value)

    def decode_delta_lists(self, data, byte_off, int_off, out, lo: int, hi: int) -> int:
        """Lists [lo, hi) of a batch, one reference decode_delta_stream per
        list (prev 0); returns the number of lists not OK.  Releases the GIL."""
        return int(self.L.mvbref_decode_delta_lists(_p(data), _p(byte_off), _p(int_off), _p(out), lo, hi))

    def decode_delta_stream(self, data, count: int, prev: int, mode: int = STRICT, path: int = 0,
                            handoff: int = 0, out: Optional[np.ndarray] = None):
        src = _u8(data)
        out = np.zeros(max(count, 0) + 4, np.uint32) if out is None else out
        r = self.L.mvbref_decode_delta_stream(_p(src), src.size, count, prev & 0xFFFFFFFF, _p(out), mode,
                                              path, handoff)
        return r.tuple(), out[:count]
