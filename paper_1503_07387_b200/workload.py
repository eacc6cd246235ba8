"""Seeded synthetic inputs for the BASELINE.json configs.

The reference measures on ClueWeb09 posting lists, which
are not available; BASELINE.json's synthetic configs stand in for them with
the shapes, sizes and value distributions stated there.  Generation is host
C++ (csrc/workload.cpp, libstdc++ mt19937 / mt19937_64); config 1 is exactly
the reference tests' mixed_values(2^24, 42).  Every Workload carries the
encoded bytes and its ground truth (the values, or the gaps whose mod-2^32
prefix sum is the expected delta output).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib


def _p(a: np.ndarray) -> Optional[int]:
    return a.ctypes.data if a.size else None


def encode(values: np.ndarray) -> np.ndarray:
    """Canonical VByte encoding (multi-threaded host encoder)."""
    v = np.ascontiguousarray(values, dtype=np.uint32)
    w = _lib.workload_lib()
    n = w.mvbw_encoded_length(_p(v), v.size)
    out = np.empty(n, np.uint8)
    w.mvbw_encode(_p(v), v.size, _p(out))
    return out


@dataclass
class Workload:
    name: str
    delta: bool
    values: np.ndarray            # uint32: decoded values (plain) or gaps (delta)
    encoded: np.ndarray           # uint8 VByte stream
    prev: int = 0
    # batched lists (config 3): per-list byte offsets (lists+1) and int offsets (lists+1)
    byte_offsets: Optional[np.ndarray] = None
    int_offsets: Optional[np.ndarray] = None
    meta: dict = field(default_factory=dict)

    @property
    def count(self) -> int:
        return int(self.values.size)

    @property
    def bytes_per_int(self) -> float:
        return self.encoded.size / max(1, self.count)

    def expected(self) -> np.ndarray:
        """Ground-truth decode output (mod-2^32 prefix sums for delta)."""
        if not self.delta:
            return self.values
        if self.int_offsets is None:
            c = np.cumsum(self.values, dtype=np.uint64) + np.uint64(self.prev)
            return (c & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        out = np.empty_like(self.values)
        io = self.int_offsets
        for i in range(io.size - 1):
            seg = self.values[io[i]:io[i + 1]]
            out[io[i]:io[i + 1]] = (np.cumsum(seg, dtype=np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        return out


def mixed_values(n: int, seed: int) -> np.ndarray:
    """The reference tests' mixed_values (decode_test.cpp:22-34)."""
    v = np.empty(int(n), np.uint32)
    _lib.workload_lib().mvbw_mixed_values(_p(v), v.size, int(seed))
    return v


def mixture(n: int, seed: int, p: float, b1, b2) -> np.ndarray:
    v = np.empty(int(n), np.uint32)
    _lib.workload_lib().mvbw_mixture(_p(v), v.size, int(seed), float(p), b1[0], b1[1], b2[0], b2[1])
    return v


def config1(n: int = 1 << 24, seed: int = 42) -> Workload:
    """Plain decode; length U{1..5}, value uniform in its length bracket."""
    v = mixed_values(n, seed)
    return Workload("c1_plain_mixed", False, v, encode(v), meta={"seed": seed, "n": n})


def config2(n: int = 1 << 24, seed: int = 7) -> Workload:
    """Delta decode of one list; gaps 50% U[1,2^7) / 50% U[2^7,2^14), prev 0.
    The gap sum exceeds 2^32 (SURVEY.md §0 finding 3), so gaps are encoded
    directly and outputs are mod-2^32 prefix sums."""
    g = mixture(n, seed, 0.5, (1, 127), (128, 16383))
    return Workload("c2_delta_1B2B", True, g, encode(g), prev=0, meta={"seed": seed, "n": n})


def config4(n: int = 1 << 30, seed: int = 3) -> Workload:
    """Large delta stream; gaps 99% 1+Geom(1/3) (mean 3), 1% U[2^14,2^21)."""
    g = np.empty(int(n), np.uint32)
    _lib.workload_lib().mvbw_geometric_gaps(_p(g), g.size, int(seed), 1.0 / 3.0, 0.01, 1 << 14, (1 << 21) - 1)
    return Workload("c4_delta_geometric", True, g, encode(g), prev=0, meta={"seed": seed, "n": n})


C5_POINTS = ("all1", "all5", "p10", "p25", "p50", "p75", "p90")


def config5(point: str, delta: bool = False, n: int = 1 << 26, seed: int = 5) -> Workload:
    """Byte-length sweep point: all-1B, all-5B, or 1B/2B mixture P(2B)=p."""
    if point == "all1":
        v = mixture(n, seed, 0.0, (0, 127), (0, 127))
    elif point == "all5":
        v = mixture(n, seed, 0.0, (1 << 28, 0xFFFFFFFF), (1 << 28, 0xFFFFFFFF))
    else:
        p = int(point[1:]) / 100.0
        v = mixture(n, seed, p, (0, 127), (128, 16383))
    return Workload(f"c5_{'delta' if delta else 'plain'}_{point}", delta, v, encode(v), prev=0,
                    meta={"seed": seed, "n": n, "point": point})


def config3(lists: int = 65536, seed: int = 11, universe: int = 1 << 25,
            min_len: int = 16, max_len: int = 65536) -> Workload:
    """Batched posting lists: log-uniform lengths, clustered sorted ids, each
    list delta-encoded from 0 (runner.cpp:28-61) and concatenated."""
    w = _lib.workload_lib()
    lengths = np.empty(lists, np.uint32)
    w.mvbw_loguniform_lengths(_p(lengths), lists, int(seed), min_len, max_len)
    int_off = np.zeros(lists + 1, np.uint64)
    np.cumsum(lengths, out=int_off[1:])
    ids = np.empty(int(int_off[-1]), np.uint32)
    w.mvbw_clustered_lists(_p(ids), _p(lengths), _p(int_off), lists, int(seed), int(universe))
    gaps = np.empty_like(ids)
    w.mvbw_delta_lists(_p(ids), _p(int_off), lists, _p(gaps))
    enc = encode(gaps)
    # per-list byte offsets from per-int encoded sizes
    sizes = (1 + (gaps >= 1 << 7).astype(np.uint8) + (gaps >= 1 << 14) + (gaps >= 1 << 21) + (gaps >= 1 << 28))
    byte_cum = np.zeros(ids.size + 1, np.uint64)
    np.cumsum(sizes, dtype=np.uint64, out=byte_cum[1:])
    byte_off = byte_cum[int_off.astype(np.int64)]
    return Workload("c3_batched_lists", True, gaps, enc, prev=0, byte_offsets=byte_off,
                    int_offsets=int_off, meta={"seed": seed, "lists": lists, "universe": universe})


CONFIGS = {
    "c1": config1,
    "c2": config2,
    "c3": config3,
    "c4": config4,
}
