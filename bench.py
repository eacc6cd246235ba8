"""Benchmark of the B200 VByte decoder (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

A step is one decode of one synthetic stream.  The default is BASELINE.json
configs[3] (c4): delta decode of 2^30 gaps (geometric, mean 3, plus 1% of
3-byte gaps), the largest config that fits one GPU and the one the north
star's scaling target names.  `value` is decoded integers per second over
all ranks with the input resident in HBM (the input, 1.1 GB, and the output,
4.3 GB, are both far larger than the 126 MB L2); `e2e` is the same metric
through the host-pointer C-ABI drop-in (mvb_decode_delta_stream) with pinned
host buffers, H2D and D2H inside the timed region.

Multi-GPU (torchrun): c4 is split by byte range across the ranks (strong
scaling): per step a totals pass over the shard, one NCCL all-gather of a
16-byte record per rank, a carry kernel and the decode, all on-stream.
c1/c2/c5 run independent replicas per rank (weak scaling, no data-path
collective); c3 partitions the lists into contiguous ranges
balanced by compressed bytes (weak in bytes per rank, no collective).
Timing is CUDA events with barrier + synchronize on both sides and the max
over ranks.

--impl reference times the reference's own CPU decoder (oracle/_ref, the
unmodified reference library built from its sources) on this host's cores,
on the same config: one stream per thread, as many threads as the host has,
each decoding its own replica of a bounded sample of the same stream (the
reference cannot split one stream).  Its input bytes come from
the reference's own encoder; the values are generated in a child process so
that the timed process maps no library of ours.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decoded uint32 integers/sec (billions) and achieved HBM GB/s vs peak"
UNIT = "Gint/s"


NOMINAL_HBM_GBS = 8000.0  # B200 nominal HBM3e bandwidth (report both denominators)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_ncu_traffic(workload):
    """DRAM bytes (read + write) per launch of the decode kernel on this
    workload, from the committed ncu --set full summary of the current build
    (profiles/r02/ncu_traffic.json; null if the workload was not captured)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "ncu_traffic.json")) as f:
            d = json.load(f)
        v = d.get(workload)
        return float(v["dram_bytes_per_launch"]) if v is not None else None
    except Exception:
        return None


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def config_dict(name, count, in_bytes, bytes_per_int, delta, world, lists=None):
    """The `config` object of both arms (identical for the same config and N)."""
    d = {"workload": name, "n": int(count), "in_bytes": int(in_bytes), "bytes_per_int": round(float(bytes_per_int), 4),
         "delta": bool(delta)}
    if lists is not None:
        d["lists"] = int(lists)
    if name.startswith("c4"):
        d["parallelism"] = f"byte-range shards x{world}" if world > 1 else "single"
    elif lists is not None:
        d["parallelism"] = f"list ranges x{world}" if world > 1 else "single"
    else:
        d["parallelism"] = f"replicas x{world}" if world > 1 else "single"
    total = int(in_bytes) + 4 * int(count)
    d["l2"] = (f"inputs larger than L2 ({total / 1e6:.0f} MB in + out > 126 MB)" if total > 4 * 126_000_000 else
               f"rotating 4 input/output sets ({4 * total / 1e6:.0f} MB > 126 MB L2)")
    return d


def make_workload(name):
    from paper_1503_07387_b200 import workload as W

    if name == "c1":
        return W.config1()
    if name == "c2":
        return W.config2()
    if name == "c3":
        return W.config3()
    if name == "c4":
        return W.config4()
    if name.startswith("c5"):
        # c5_<point>[_delta]
        parts = name.split("_")
        return W.config5(parts[1], delta=len(parts) > 2 and parts[2] == "delta")
    raise SystemExit(f"unknown config {name}")


class ClockSampler:
    """NVML sampling of SM clock and clock-event reasons during the timed region."""

    BAD = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
           "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.BAD.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_reference_rate(w, seconds, threads, gate=True):
    """Reference library (oracle/_ref) decode of the workload stream on `threads`
    host threads, each decoding its own replica; returns (ints/s, reps)."""
    from oracle import RefLib

    ref = RefLib()
    enc = np.ascontiguousarray(w.encoded)
    outs = [np.empty(w.count + 16, np.uint32) for _ in range(threads)]
    counts = [0] * threads
    stop_at = [0.0]

    def work(i):
        n = 0
        while True:
            if w.delta:
                r, _ = ref.decode_delta_stream(enc, w.count, w.prev, out=outs[i])
            else:
                r, _ = ref.decode_stream(enc, w.count, out=outs[i])
            assert r[0] == 0 and r[1] == w.count
            n += 1
            if time.perf_counter() >= stop_at[0] and n >= 1:
                break
        counts[i] = n

    if gate:  # correctness gate (runner.cpp:147-165): reference output equals ground truth
        if w.delta:
            r, o = ref.decode_delta_stream(enc, w.count, w.prev, out=outs[0])
        else:
            r, o = ref.decode_stream(enc, w.count, out=outs[0])
        assert np.array_equal(o, w.expected()), "reference decode disagrees with ground truth"
    t0 = time.perf_counter()
    stop_at[0] = t0 + seconds
    ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    dt = time.perf_counter() - t0
    return sum(counts) * w.count / dt, sum(counts)


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


SAMPLE_INTS = 1 << 26  # reference arm / cpu_baseline sample of a long stream: its first 2^26 integers


def emit_values(cfg: str) -> None:
    """(child process of the reference arm) Generate workload `cfg` and write a
    JSON header line plus the raw sample: the first SAMPLE_INTS values (or gaps)
    of a stream, or every list's gaps and the int offsets of a batch."""
    w = make_workload(cfg)
    lists = None if w.int_offsets is None else int(w.int_offsets.size - 1)
    k = w.count if lists is not None else min(w.count, SAMPLE_INTS)
    h = {"name": w.name, "count": w.count, "in_bytes": int(w.encoded.size), "bytes_per_int": w.bytes_per_int,
         "delta": w.delta, "prev": int(w.prev), "k": int(k), "lists": lists}
    out = sys.stdout.buffer
    out.write((json.dumps(h) + "\n").encode())
    out.write(np.ascontiguousarray(w.values[:k], dtype=np.uint32).tobytes())
    if lists is not None:
        out.write(np.ascontiguousarray(w.int_offsets, dtype=np.uint64).tobytes())
    out.flush()


def reference_input(cfg: str):
    """The reference arm's input: values from a child process (so this process
    maps no library of ours), bytes from the reference's own encoder."""
    import subprocess

    from oracle import RefLib

    p = subprocess.run([sys.executable, os.path.abspath(__file__), "--emit-values", cfg], capture_output=True,
                       check=True)
    nl = p.stdout.index(b"\n")
    h = json.loads(p.stdout[:nl])
    body = memoryview(p.stdout)[nl + 1:]
    k = h["k"]
    vals = np.frombuffer(body[:4 * k], dtype=np.uint32)
    io = None
    if h["lists"] is not None:
        io = np.frombuffer(body[4 * k:4 * k + 8 * (h["lists"] + 1)], dtype=np.uint64)
    ref = RefLib()
    enc = ref.encode_sequence(vals)  # VByte is per integer: the lists' concatenation is one stream
    bo = None
    if io is not None:
        sizes = (1 + (vals >= 1 << 7).astype(np.uint8) + (vals >= 1 << 14) + (vals >= 1 << 21) + (vals >= 1 << 28))
        cum = np.zeros(vals.size + 1, np.uint64)
        np.cumsum(sizes, dtype=np.uint64, out=cum[1:])
        bo = cum[io.astype(np.int64)]
    return h, vals, enc, bo, io


def run_reference(args):
    world, rank, _ = dist_setup(args)
    if rank != 0:
        return
    from oracle import RefLib

    ref = RefLib()
    h, vals, enc, bo, io = reference_input(args.config)
    threads = os.cpu_count() or 1
    model = cpu_model()
    cfg = config_dict(h["name"], h["count"], h["in_bytes"], h["bytes_per_int"], h["delta"], args.gpus, h["lists"])
    if io is not None:  # c3: lists split over all host threads, each step a bounded sample
        out = np.empty(vals.size + 16, np.uint32)
        n = io.size - 1
        cuts = np.linspace(0, n, threads + 1).astype(np.int64)
        assert ref.decode_delta_lists(enc, bo, io, out, 0, n) == 0
        exp_ok = all(np.array_equal(out[int(io[i]):int(io[i]) + 3],
                                    np.cumsum(vals[int(io[i]):int(io[i]) + 3], dtype=np.uint64).astype(np.uint32))
                     for i in range(0, n, max(1, n // 64)))
        assert exp_ok, "reference list decode disagrees with ground truth"

        def step(seconds):
            done, ints = [0] * threads, [0] * threads
            stop_at = time.perf_counter() + seconds

            def work(i):
                lo, hi = int(cuts[i]), int(cuts[i + 1])
                while True:
                    assert ref.decode_delta_lists(enc, bo, io, out, lo, hi) == 0
                    ints[i] += int(io[hi] - io[lo])
                    if time.perf_counter() >= stop_at:
                        break

            t0 = time.perf_counter()
            ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
            for t in ths:
                t.start()
            for t in ths:
                t.join()
            return sum(ints), time.perf_counter() - t0

        for _ in range(args.warmup):
            step(0.0)
        t_steps, n_ints = [], 0
        for _ in range(args.steps):
            k, dt = step(0.5)
            n_ints += k
            t_steps.append(dt)
        value = n_ints / sum(t_steps) / 1e9
        sample = (f"each step: ~0.5 s of list decodes (mvb::decode_delta_stream per list, runner.cpp decode_list), "
                  f"lists split over {threads} threads")
    else:
        # One stream: the reference decodes a stream on one thread and has no way
        # to split it (runner.cpp:174-196 times one thread per
        # stream), so the arm times one thread on the stream's first
        # SAMPLE_INTS integers.  The aggregate of `threads` threads each decoding
        # its own replica -- a different workload, many streams -- is reported
        # beside it (replicas_all_threads).
        k = vals.size
        outs = [np.empty(k + 16, np.uint32) for _ in range(threads)]
        dec = (lambda o: ref.decode_delta_stream(enc, k, h["prev"], out=o)) if h["delta"] else \
            (lambda o: ref.decode_stream(enc, k, out=o))
        r, o = dec(outs[0])  # correctness gate (runner.cpp:147-165)
        exp = (np.cumsum(vals, dtype=np.uint64) + np.uint64(h["prev"])).astype(np.uint32) if h["delta"] else vals
        assert r[0] == 0 and r[1] == k and np.array_equal(o, exp), "reference decode disagrees with ground truth"

        def step(nthreads):
            def work(i):
                r, _ = dec(outs[i])
                assert r[0] == 0

            t0 = time.perf_counter()
            ths = [threading.Thread(target=work, args=(i,)) for i in range(nthreads)]
            for t in ths:
                t.start()
            for t in ths:
                t.join()
            return time.perf_counter() - t0

        for _ in range(args.warmup):
            step(1)
        t_steps = [step(1) for _ in range(args.steps)]
        value = k * args.steps / sum(t_steps) / 1e9
        for _ in range(max(1, args.warmup)):
            step(threads)
        t_rep = [step(threads) for _ in range(args.steps)]
        replicas = {"value": k * threads * args.steps / sum(t_rep) / 1e9, "unit": UNIT, "threads": threads,
                    "sample": f"each step: {threads} threads x 1 decode of their own replica of the sample "
                              "(many independent streams: not this config's one stream)"}
        sample = (f"each step: 1 thread x 1 decode of the first {k} integers of the {h['name']} stream "
                  f"(reference encoder's bytes) with mvb::decode{'_delta' if h['delta'] else ''}_stream "
                  "(SSE masked path); one stream cannot be split across threads")
        threads = 1
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(t_steps) / args.steps,
        "higher_is_better": True, "scaling": "strong" if h["name"].startswith("c4") else "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample,
                         "cpu_model": model},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if io is None:
        line["replicas_all_threads"] = replicas
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1503_07387_b200 import _lib, mvb

    world, rank, local = dist_setup(args)
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)

    w = make_workload(args.config)
    count, in_len = w.count, int(w.encoded.size)
    R = 4  # rotating buffer sets
    srcs = [torch.from_numpy(w.encoded).to(dev) for _ in range(R)]
    outs = [torch.empty(count, dtype=torch.int32, device=dev) for _ in range(R)]
    dec = mvb.Decoder(dev, capacity_bytes=in_len)
    expected = torch.from_numpy(w.expected().view(np.int32)).to(dev)
    stream = torch.cuda.current_stream(dev)

    def step(i):
        k = i % R
        if w.delta:
            dec.decode_delta(srcs[k], count, w.prev, outs[k])
        else:
            dec.decode(srcs[k], count, outs[k])

    # correctness gate
    for k in range(R):
        step(k)
    r = dec.result()
    assert int(r.status) == 0 and r.values_written == count and r.bytes_consumed == in_len, r
    for k in range(R):
        assert torch.equal(outs[k], expected), "GPU decode disagrees with ground truth"
    del expected

    # warm-up, including a >= 1 s sustained pre-roll so clocks settle
    for i in range(max(args.warmup, 3)):
        step(i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    i = 0
    while time.perf_counter() - t0 < args.preroll:
        for _ in range(64):
            step(i)
            i += 1
        torch.cuda.synchronize()

    # the timed region holds only the decodes: events between them would cost ~5 us
    # each (they break the back-to-back launch of kernel A behind the previous
    # kernel B), so a decode's duration is the region's time / steps
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        start = torch.cuda.Event(enable_timing=True)
        stop = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for s in range(args.steps):
            step(s)
        stop.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = start.elapsed_time(stop)
    kern_ms = [total_ms / args.steps]
    r = dec.result()
    assert int(r.status) == 0 and r.values_written == count

    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = world * count * args.steps / (total_ms / 1e3) / 1e9

    # roofline of the decode kernel: algorithmic bytes = input + 4 B per int
    alg_bytes = in_len + 4 * count
    avg_kernel_s = statistics.mean(kern_ms) / 1e3
    achieved = alg_bytes / avg_kernel_s / 1e9
    peak, peak_kind = load_peaks()
    traffic = load_ncu_traffic(w.name)

    # end to end through the host C-ABI drop-in with pinned host buffers
    h_in = torch.from_numpy(w.encoded).pin_memory()
    h_out = torch.empty(count, dtype=torch.int32).pin_memory()
    L = _lib.lib()
    res = _lib.MvbResult()

    def e2e_call():
        if w.delta:
            rc = L.mvb_decode_delta_stream(h_in.data_ptr(), in_len, count, w.prev, h_out.data_ptr(), 0,
                                           ctypes.byref(res))
        else:
            rc = L.mvb_decode_stream(h_in.data_ptr(), in_len, count, h_out.data_ptr(), 0, ctypes.byref(res))
        assert rc == 0 and res.values_written == count, (rc, res.values_written)

    for _ in range(3):
        e2e_call()
    assert np.array_equal(h_out.numpy().view(np.uint32), w.expected()), "e2e output mismatch"
    if world > 1:
        dist.barrier()
    e_steps = max(3, min(args.steps, 50))
    t0 = time.perf_counter()
    for _ in range(e_steps):
        e2e_call()
    e_dt = time.perf_counter() - t0
    et = torch.tensor([e_dt], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_value = world * count * e_steps / float(et.item()) / 1e9

    cpu = None
    if rank == 0 and world == 1 and args.cpu_seconds > 0:
        try:
            rate, reps = cpu_reference_rate(w, args.cpu_seconds, 1)
            cpu = {"value": rate / 1e9, "unit": UNIT, "cores": 1, "kind": "reference", "cpu_model": cpu_model(),
                   "sample": f"{reps} full decodes of the {w.name} stream ({count} ints) by the reference "
                             f"library's decode{'_delta' if w.delta else ''}_stream (SSE masked path), 1 thread, "
                             f"~{args.cpu_seconds:.0f} s"}
        except Exception as e:  # reference build missing on this host
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": config_dict(w.name, count, in_len, w.bytes_per_int, w.delta, world),
            "hbm_gbs": achieved,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac_of_nominal_8000": achieved / NOMINAL_HBM_GBS,
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "alg_bytes_per_launch": alg_bytes, "kernel_ms_avg": statistics.mean(kern_ms),
                         "kernel_ms_note": "decode (kernels A + B) time = timed region / steps, launched "
                                           "back to back on the current stream"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": in_len,
                    "d2h_bytes_per_step": 4 * count + ctypes.sizeof(_lib.MvbResult),
                    "api": "mvb_decode_delta_stream (host pointers, pinned)" if w.delta else
                           "mvb_decode_stream (host pointers, pinned)"},
            "gpu_launches": args.steps * _lib.kernels_per_decode(0),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _check_shard_values(torch, dev, vals, gaps, offset, prev):
    """Device-side check of a shard's delta output against the ground-truth
    gaps: out[i] = prev + gaps[0] + ... + gaps[offset + i] (mod 2^32)."""
    carry = (prev + int(gaps[:offset].astype(np.uint64).sum())) & 0xFFFFFFFF
    step = 1 << 26
    for a in range(0, vals.numel(), step):
        g = torch.from_numpy(gaps[offset + a: offset + a + min(step, vals.numel() - a)].astype(np.int64)).to(dev)
        exp = (torch.cumsum(g, 0) + carry) & 0xFFFFFFFF
        got = vals[a:a + g.numel()].to(torch.int64) & 0xFFFFFFFF
        if not torch.equal(got, exp):
            return False
        carry = int(exp[-1].item())
    return True


def run_sharded(args):
    """Config 4: one 2^30-integer delta stream split by byte range across the
    ranks (strong scaling).  A step is one pass of
    DeviceShard.run() on every rank: totals pre-pass, NCCL all-gather of a
    16-byte record, carry kernel, decode with the device-resident carry."""
    import torch
    import torch.distributed as dist

    from paper_1503_07387_b200 import shard as S

    world, rank, local = dist_setup(args)
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)

    w = make_workload(args.config)
    L = int(w.encoded.size)
    lo, hi = S.local_range(L, world, rank)
    h_buf = torch.from_numpy(w.encoded[lo:hi]).pin_memory()
    buf = h_buf.to(dev)
    sh = S.DeviceShard(buf, lo, L, w.delta, w.prev, world, rank)
    stream = torch.cuda.current_stream(dev)

    # correctness gate: whole-stream result and this rank's slice of the values
    sh.run()
    off, vals, glob = sh.result()
    assert glob == (0, w.count, L), glob
    if w.delta:
        assert _check_shard_values(torch, dev, vals, w.values, off, w.prev), "sharded decode mismatch"
    else:
        assert torch.equal(vals, torch.from_numpy(w.values[off:off + vals.numel()].view(np.int32)).to(dev))
    n_local = int(vals.numel())
    del vals

    for _ in range(max(args.warmup, 3)):
        sh.run()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < args.preroll:
        for _ in range(8):
            sh.run()
        torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        start = torch.cuda.Event(enable_timing=True)
        stop = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for s in range(args.steps):
            sh.prepass()
            if w.delta and world > 1:
                sh.exchange()
            ev[s][0].record(stream)
            sh.decode()
            ev[s][1].record(stream)
        stop.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = start.elapsed_time(stop)
    kern_ms = [a.elapsed_time(b) for a, b in ev]
    _, _, glob = sh.result()
    assert glob == (0, w.count, L), glob
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = w.count * args.steps / (total_ms / 1e3) / 1e9

    shard_bytes = sh.bound
    alg_bytes = shard_bytes + 4 * n_local
    achieved = alg_bytes / (statistics.mean(kern_ms) / 1e3) / 1e9
    peak, peak_kind = load_peaks()

    # end to end: H2D of this rank's byte range from pinned memory, the pass,
    # D2H of its decoded integers, every step.  One GPU: the whole stream through
    # the host-pointer drop-in (mvb_decode_delta_stream, pipelined chunks)
    h_out = torch.empty(max(sh.bound, 1) if world > 1 else max(w.count, 1), dtype=torch.int32).pin_memory()
    from paper_1503_07387_b200 import _lib
    Lh = _lib.lib()
    e2e_api = "DeviceShard.run (pre-pass, all-gather, carry, decode) with pinned H2D/D2H"
    if world == 1:
        e2e_api = "mvb_decode_delta_stream (host pointers, pinned, pipelined chunks)"
        res_h = _lib.MvbResult()

    def e2e_step():
        if world == 1:
            rc = Lh.mvb_decode_delta_stream(h_buf.data_ptr(), L, w.count, w.prev, h_out.data_ptr(), 0,
                                            ctypes.byref(res_h))
            assert rc == 0 and res_h.values_written == w.count, (rc, res_h.values_written)
            return
        buf.copy_(h_buf, non_blocking=True)
        sh.run()
        h_out[:n_local].copy_(sh.out[:n_local], non_blocking=True)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e_steps = max(3, min(args.steps, 20))
    t0 = time.perf_counter()
    for _ in range(e_steps):
        e2e_step()
    torch.cuda.synchronize()
    e_dt = time.perf_counter() - t0
    et = torch.tensor([e_dt], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_value = w.count * e_steps / float(et.item()) / 1e9

    cpu = None
    if rank == 0 and world == 1 and args.cpu_seconds > 0:
        try:
            rate, reps, sample = cpu_reference_sample(w, args.cpu_seconds, 1)
            cpu = {"value": rate / 1e9, "unit": UNIT, "cores": 1, "kind": "reference", "sample": sample,
                   "cpu_model": cpu_model()}
        except Exception as e:
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": config_dict(w.name, w.count, L, w.bytes_per_int, w.delta, world),
            "hbm_gbs": achieved,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac_of_nominal_8000": achieved / NOMINAL_HBM_GBS,
                         "frac": achieved / peak, "traffic": load_ncu_traffic(w.name), "peak_kind": peak_kind,
                         "alg_bytes_per_launch": alg_bytes, "kernel_ms_avg": statistics.mean(kern_ms),
                         "kernel_ms_min": min(kern_ms), "kernel": "decode of rank 0's shard"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h_buf.numel()),
                    "d2h_bytes_per_step": 4 * (n_local if world > 1 else w.count), "api": e2e_api},
            "gpu_launches": args.steps * sh.launches_per_pass,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_lists_rate(w, seconds, threads, gate=True):
    """Reference decode of the c3 lists: each host thread decodes its own
    share of the lists with one mvb::decode_delta_stream per list (the
    reference's runner.cpp decode_list loop), repeating until `seconds`
    elapse; returns (ints/s, list decodes done, ints decoded)."""
    from oracle import RefLib

    ref = RefLib()
    enc = np.ascontiguousarray(w.encoded)
    bo = np.ascontiguousarray(w.byte_offsets.astype(np.uint64))
    io = np.ascontiguousarray(w.int_offsets.astype(np.uint64))
    out = np.empty(w.count + 16, np.uint32)
    n = bo.size - 1
    cuts = np.linspace(0, n, threads + 1).astype(np.int64)
    if gate:
        assert ref.decode_delta_lists(enc, bo, io, out, 0, n) == 0
        assert np.array_equal(out[:w.count], w.expected()), "reference list decode disagrees with ground truth"
    done = [0] * threads
    ints = [0] * threads
    stop_at = [time.perf_counter() + seconds]

    def work(i):
        lo, hi = int(cuts[i]), int(cuts[i + 1])
        while True:
            assert ref.decode_delta_lists(enc, bo, io, out, lo, hi) == 0
            done[i] += hi - lo
            ints[i] += int(io[hi] - io[lo])
            if time.perf_counter() >= stop_at[0]:
                break

    t0 = time.perf_counter()
    ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    dt = time.perf_counter() - t0
    return sum(ints) / dt, sum(done), sum(ints)


def run_lists(args):
    """Config 3: 65,536 independent delta-coded posting lists decoded in one
    launch (mvb_decode_delta_lists_device, one warp per list, longest first).
    A step decodes the whole batch.  Multi-GPU: each rank decodes a contiguous
    range of lists balanced by compressed bytes (shard.list_ranges; SURVEY.md
    §8e: independent units, no exchange) -- the batch is split, not replicated."""
    import torch
    import torch.distributed as dist

    from paper_1503_07387_b200 import _lib, mvb
    from paper_1503_07387_b200.shard import list_ranges

    world, rank, local = dist_setup(args)
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    w = make_workload(args.config)
    n_all = w.byte_offsets.size - 1
    cuts = list_ranges(w.byte_offsets, world)
    l0, l1 = cuts[rank], cuts[rank + 1]
    bo_all = w.byte_offsets.astype(np.int64)
    io_all = w.int_offsets.astype(np.int64)
    b0, b1, i0, i1 = int(bo_all[l0]), int(bo_all[l1]), int(io_all[l0]), int(io_all[l1])
    n_lists, n_ints, n_bytes = l1 - l0, i1 - i0, b1 - b0
    bo_r = (bo_all[l0:l1 + 1] - b0).astype(np.uint64)
    io_r = (io_all[l0:l1 + 1] - i0).astype(np.uint64)
    lens = np.diff(bo_r.astype(np.int64))
    order_np = np.argsort(-lens, kind="stable").astype(np.uint32)
    h_in = torch.from_numpy(np.ascontiguousarray(w.encoded[b0:b1])).pin_memory()
    h_bo = torch.from_numpy(bo_r.view(np.int64)).pin_memory()
    h_io = torch.from_numpy(io_r.view(np.int64)).pin_memory()
    src, bo, io = h_in.to(dev), h_bo.to(dev), h_io.to(dev)
    order = torch.from_numpy(order_np.view(np.int32)).to(dev)
    out = torch.empty(max(n_ints, 1), dtype=torch.int32, device=dev)
    res = torch.zeros(max(n_lists, 1) * 3, dtype=torch.int64, device=dev)
    d = mvb.Decoder(dev, 1 << 12)
    stream = torch.cuda.current_stream(dev)
    expected = w.expected()[i0:i1]

    def step():
        d.decode_lists(src, bo, io, out[:n_ints], order=order, results=res, delta=True)

    step()
    torch.cuda.synchronize()
    rr = res.cpu().numpy().reshape(-1, 3)[:n_lists]
    assert (rr[:, 0] == 0).all() and (rr[:, 1] == np.diff(io_r.astype(np.int64))).all(), "list results"
    assert torch.equal(out[:n_ints], torch.from_numpy(expected.view(np.int32)).to(dev)), "batched list decode mismatch"
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        start = torch.cuda.Event(enable_timing=True)
        stop = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for s_ in range(args.steps):
            ev[s_][0].record(stream)
            step()
            ev[s_][1].record(stream)
        stop.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = start.elapsed_time(stop)
    kern_ms = [a.elapsed_time(b) for a, b in ev]
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = w.count * args.steps / (total_ms / 1e3) / 1e9  # every rank's lists: the whole batch per step
    meta = (n_lists + 1) * 16 + n_lists * 4 + n_lists * 24  # offsets, order, results
    alg_bytes = n_bytes + 4 * n_ints + meta
    achieved = alg_bytes / (statistics.mean(kern_ms) / 1e3) / 1e9
    peak, peak_kind = load_peaks()

    # end to end through the host-pointer batched entry (mvb_decode_delta_lists:
    # pinned buffers; this rank's bytes, offsets and values cross PCIe every
    # call, in pipelined sub-batches)
    h_out = torch.empty(max(n_ints, 1), dtype=torch.int32).pin_memory()
    Lh = _lib.lib()

    def e2e_step():
        rc = Lh.mvb_decode_delta_lists(h_in.data_ptr(), n_bytes, h_bo.data_ptr(), h_io.data_ptr(), None, n_lists,
                                       h_out.data_ptr(), 0, None)
        assert rc == 0, rc

    e2e_step()
    assert np.array_equal(h_out.numpy()[:n_ints].view(np.uint32), expected), "e2e output mismatch"
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e_steps = max(3, min(args.steps, 10))
    t0 = time.perf_counter()
    for _ in range(e_steps):
        e2e_step()
    torch.cuda.synchronize()
    et = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_value = w.count * e_steps / float(et.item()) / 1e9

    cpu = None
    if rank == 0 and world == 1 and args.cpu_seconds > 0:
        try:
            threads = os.cpu_count() or 1
            rate, lists_done, ints_done = cpu_lists_rate(w, args.cpu_seconds, threads)
            cpu = {"value": rate / 1e9, "unit": UNIT, "cores": threads, "kind": "reference", "cpu_model": cpu_model(),
                   "sample": f"{lists_done} list decodes ({ints_done} ints) of the {w.name} batch by the reference "
                             f"library's decode_delta_stream, one call per list (runner.cpp decode_list), lists "
                             f"split over {threads} host threads, ~{args.cpu_seconds:.0f} s"}
        except Exception as e:
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": config_dict(w.name, w.count, int(w.encoded.size), w.bytes_per_int, True, world, n_all),
            "hbm_gbs": achieved,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac_of_nominal_8000": achieved / NOMINAL_HBM_GBS, "frac": achieved / peak,
                         "traffic": load_ncu_traffic(w.name), "peak_kind": peak_kind, "alg_bytes_per_launch": alg_bytes,
                         "kernel_ms_avg": statistics.mean(kern_ms), "kernel_ms_min": min(kern_ms),
                         "kernel": "vbyte_lists_decode_units (one launch per batch; rank 0's list range)"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": n_bytes + 2 * (n_lists + 1) * 8,
                    "d2h_bytes_per_step": 4 * n_ints,
                    "api": "mvb_decode_delta_lists (host pointers, pinned, pipelined sub-batches)"},
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_reference_sample(w, seconds, threads):
    """Reference decode rate on a bounded prefix of a large stream (2^26
    integers, the reference's l1-style chunk of the same bytes)."""
    from paper_1503_07387_b200 import workload as W

    k = min(w.count, 1 << 26)
    sub = W.Workload(w.name, w.delta, w.values[:k], w.encoded[:int(W.encode(w.values[:k]).size)], prev=w.prev)
    rate, reps = cpu_reference_rate(sub, seconds, threads)
    return rate, reps, (f"{reps} decodes of the first {k} integers of the {w.name} stream by the reference "
                        f"library's decode{'_delta' if w.delta else ''}_stream (SSE masked path), "
                        f"{threads} thread(s), ~{seconds:.0f} s")


def run_csv(args):
    """Reference-schema CSV (K,bits_per_int,scheme,mis,ratio_vs_scalar,
    buffer_mode): `cuda` rows from the batched GPU decode
    (paper_1503_07387_b200/bench_csv.py) next to the reference library's own
    `scalar` and `masked` rows (oracle/_ref, the CPU leg), l1 (4096-integer
    buffer) and full modes, timed like runner.cpp:174-196."""
    from oracle import RefLib
    from paper_1503_07387_b200 import bench_csv as B
    from paper_1503_07387_b200 import mvb

    ref = RefLib()
    rows = []
    for k in range(args.k_min, args.k_max + 1):
        bufs = [mvb.encode_deltas(ids) for ids in B.group_lists(k, args.lists, args.seed)]
        ints = sum(b.count for b in bufs)
        bits = 8.0 * sum(b.bytes.size for b in bufs) / ints
        out = np.zeros(max(max(b.count for b in bufs), 4096) + 16, np.uint32)
        for scheme in ("scalar", "masked"):
            dec = ref.decode_delta_scalar if scheme == "scalar" else ref.decode_delta_stream
            for mode in ("l1", "full"):
                def one_pass(dec=dec, mode=mode):
                    for b in bufs:
                        if mode == "full":
                            dec(b.bytes, b.count, 0, out=out)
                            continue
                        done = off = prev = 0
                        while done < b.count:  # runner.cpp:35-44 / :51-60
                            n = min(4096, b.count - done)
                            r, _ = dec(b.bytes[off:], n, prev, out=out)
                            off += r[2]
                            prev = int(out[n - 1])
                            done += n
                rows.append(B.BenchResult(k, bits, scheme, B.time_passes(one_pass, args.min_ms / 1e3, args.reps, ints,
                                                                         B.wall_timer), 0.0, mode))
    rows += B.cuda_rows(args.k_min, args.k_max, args.lists, args.seed, args.reps, args.min_ms)
    rows.sort(key=lambda r: (r.k, r.buffer_mode != "l1", r.scheme))
    B.add_ratios(rows)
    with open(args.csv, "w") as f:
        B.write_csv(f, rows)
    B.write_csv(sys.stdout, rows)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--emit-values", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--preroll", type=float, default=1.0)
    ap.add_argument("--csv", default=None, help="write the reference-schema CSV (cuda / scalar / masked rows) here")
    ap.add_argument("--k-min", type=int, default=4)
    ap.add_argument("--k-max", type=int, default=16)
    ap.add_argument("--lists", type=int, default=8)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--min-ms", type=int, default=100)
    args = ap.parse_args()
    if args.emit_values:
        emit_values(args.emit_values)
    elif args.csv:
        run_csv(args)
    elif args.impl == "reference":
        run_reference(args)
    elif args.config == "c4":
        run_sharded(args)
    elif args.config == "c3":
        run_lists(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
