"""Benchmark CSV in the reference's schema with a `cuda` scheme (SURVEY.md
§8f rank 4), so GPU results sit in the same table as the reference's
`mvb bench` output (tools/bench/csv.hpp:11, csv.cpp:40-83,
runner.cpp:108-218).  `python bench.py --csv out.csv` produces the table:
this module holds the schema, the reader/writer, the groups and the `cuda`
rows; bench.py adds the reference library's `scalar` / `masked` rows (its
CPU-baseline leg).

Rows: K (length group: lists of lengths [2^K, 2^(K+1))), bits_per_int, scheme,
mis (millions of integers decoded per second, median of `--reps`
measurements, each repeated to at least --min-ms as runner.cpp does),
ratio_vs_scalar (mis / the scalar row of the same K and buffer mode; 0 if
none), buffer_mode.  Lists are sorted distinct ids drawn uniformly from
[0, 2^25) (the reference's WorkloadSpec shape; our own seeded generator, so
the bytes differ from `mvb bench`'s), delta-encoded with encode_deltas.
`scalar` and `masked` run the reference library (oracle/_ref) on the host in
"l1" (4096-integer buffer) and "full" modes; `cuda` decodes every list of the
group in one batched launch (device-resident input, CUDA events) in "full"
mode.  Doubles are written in shortest round-trip form, like the reference.
"""
from __future__ import annotations

import statistics
import time
from dataclasses import dataclass
from typing import List

import numpy as np

CSV_HEADER = "K,bits_per_int,scheme,mis,ratio_vs_scalar,buffer_mode"


@dataclass
class BenchResult:
    k: int
    bits_per_int: float
    scheme: str
    mis: float
    ratio_vs_scalar: float
    buffer_mode: str


def format_double(x: float) -> str:
    """std::to_chars(double) without a format (csv.cpp:13-18): the shortest
    digits that round-trip, written in fixed or scientific notation,
    whichever is shorter (fixed on a tie), exponent with at least 2 digits."""
    from decimal import Decimal

    x = float(x)
    if x == 0:
        return "-0" if str(x).startswith("-") else "0"
    sign, digits, exp = Decimal(repr(x)).normalize().as_tuple()
    ds = "".join(map(str, digits))
    n = len(ds)
    if exp >= 0:
        fixed = ds + "0" * exp
    elif -exp < n:
        fixed = ds[: n + exp] + "." + ds[n + exp:]
    else:
        fixed = "0." + "0" * (-exp - n) + ds
    e10 = exp + n - 1
    sci = ds[0] + ("." + ds[1:] if n > 1 else "") + ("e-" if e10 < 0 else "e+") + f"{abs(e10):02d}"
    out = fixed if len(fixed) <= len(sci) else sci
    return ("-" if sign else "") + out


def write_csv(f, results: List[BenchResult]) -> None:
    f.write(CSV_HEADER + "\n")
    for r in results:
        f.write(f"{r.k},{format_double(r.bits_per_int)},{r.scheme},{format_double(r.mis)},"
                f"{format_double(r.ratio_vs_scalar)},{r.buffer_mode}\n")


def read_csv(f) -> List[BenchResult]:
    lines = f.read().splitlines()
    if not lines or lines[0] != CSV_HEADER:
        raise RuntimeError("read_csv: missing or unexpected header")
    out = []
    for line in lines[1:]:
        if not line:
            continue
        x = line.split(",")
        if len(x) != 6:
            raise RuntimeError("read_csv: bad row: " + line)
        out.append(BenchResult(int(x[0]), float(x[1]), x[2], float(x[3]), float(x[4]), x[5]))
    return out


def group_lists(k: int, n_lists: int, seed: int, universe: int = 1 << 25):
    rng = np.random.default_rng([seed, k])
    lists = []
    for _ in range(n_lists):
        n = int(rng.integers(1 << k, 1 << (k + 1)))
        ids = np.unique(rng.integers(0, universe, n + n // 8 + 16, dtype=np.int64))
        while ids.size < n:
            ids = np.unique(np.concatenate([ids, rng.integers(0, universe, n, dtype=np.int64)]))
        ids = np.sort(rng.choice(ids, n, replace=False)).astype(np.uint32)
        lists.append(ids)
    return lists


def time_passes(one_pass, min_s: float, reps: int, ints: int, timer) -> float:
    """runner.cpp:174-196: warm up, double passes until one measurement
    spans min_s, then the median of `reps` measurements (Mint/s)."""
    one_pass()  # warmup
    passes, seconds = 1, 0.0
    while True:
        seconds = timer(lambda: [one_pass() for _ in range(passes)])
        if seconds >= min_s:
            break
        passes *= 2
    samples = [ints * passes / seconds / 1e6]
    for _ in range(1, reps):
        samples.append(ints * passes / timer(lambda: [one_pass() for _ in range(passes)]) / 1e6)
    return statistics.median(samples)


def cuda_rows(k_min=4, k_max=16, n_lists=8, seed=42, reps=3, min_ms=100) -> List[BenchResult]:
    """`cuda` rows: every list of group K decoded in one batched launch
    (device-resident, CUDA events), after a correctness gate
    (runner.cpp:147-165)."""
    import torch

    from . import mvb

    dev = torch.device("cuda", 0)
    d = mvb.Decoder(dev, 1 << 12)
    out: List[BenchResult] = []
    for k in range(k_min, k_max + 1):
        lists = group_lists(k, n_lists, seed)
        bufs = [mvb.encode_deltas(ids) for ids in lists]
        ints = sum(b.count for b in bufs)
        bits = 8.0 * sum(b.bytes.size for b in bufs) / ints
        bo = np.zeros(len(bufs) + 1, np.uint64)
        io_ = np.zeros(len(bufs) + 1, np.uint64)
        np.cumsum([b.bytes.size for b in bufs], out=bo[1:])
        np.cumsum([b.count for b in bufs], out=io_[1:])
        src = torch.from_numpy(np.concatenate([np.asarray(b.bytes, np.uint8) for b in bufs])).to(dev)
        tbo = torch.from_numpy(bo.view(np.int64)).to(dev)
        tio = torch.from_numpy(io_.view(np.int64)).to(dev)
        dout = torch.empty(ints, dtype=torch.int32, device=dev)

        def one_pass():
            d.decode_lists(src, tbo, tio, dout, delta=True)

        def cuda_timer(fn):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            return s.elapsed_time(e) / 1e3

        one_pass()
        torch.cuda.synchronize()
        if not np.array_equal(dout.cpu().numpy().view(np.uint32), np.concatenate(lists)):
            raise RuntimeError(f"decode mismatch: scheme cuda, group K={k}")
        out.append(BenchResult(k, bits, "cuda", time_passes(one_pass, min_ms / 1e3, reps, ints, cuda_timer), 0.0,
                               "full"))
    return out


def wall_timer(fn) -> float:
    t0 = time.perf_counter()
    fn()
    return time.perf_counter() - t0


def add_ratios(results: List[BenchResult]) -> List[BenchResult]:
    """runner.cpp:209-217: mis over the scalar mis of the same (K, mode)."""
    for r in results:
        for s in results:
            if s.k == r.k and s.buffer_mode == r.buffer_mode and s.scheme == "scalar":
                r.ratio_vs_scalar = r.mis / s.mis
                break
    return results
