"""Byte-range sharded decode.

CPU: the host logic (cuts, resync, per-shard counts, result combination) runs
for W ranks against the oracle -- in-process with a threaded all-gather for
many edge cases, and across real processes over a `gloo` group.  GPU: the
totals pass (mvb_delta_totals_device) against the oracle, W virtual shards
decoded by the CUDA kernels on one device through the Python shard logic, and
the C-ABI multi-GPU entry (mvb_decode_delta_sharded) over W virtual GPUs.  Every result must equal the
whole-stream oracle decode bit for bit (values and DecodeResult).
"""
import os
import threading

import numpy as np
import pytest

from oracle import Oracle, STRICT
from paper_1503_07387_b200 import shard as S
from paper_1503_07387_b200 import workload as W

ORACLE = None


def oracle():
    global ORACLE
    if ORACLE is None:
        ORACLE = Oracle()
    return ORACLE


class OracleOps(S.ShardOps):
    """Test double for the device ops: the CPU oracle (checker only)."""

    def totals(self, shard):
        shard = np.asarray(shard, np.uint8)
        n = int((shard < 0x80).sum())
        _, vals = oracle().decode(shard, n, STRICT)
        return n, int(vals.astype(np.uint64).sum() & 0xFFFFFFFF)

    def decode(self, shard, count, prev, delta, out=None):
        if delta:
            return oracle().decode_delta(np.asarray(shard, np.uint8), count, prev, STRICT)
        return oracle().decode(np.asarray(shard, np.uint8), count, STRICT)


class ThreadGather:
    """all_gather over W threads of one process (lock-step, two barriers)."""

    def __init__(self, world):
        self.world = world
        self.slots = [None] * world
        self.bar = threading.Barrier(world)

    def for_rank(self, rank):
        def gather(rec):
            self.slots[rank] = list(rec)
            self.bar.wait()
            res = [list(r) for r in self.slots]
            self.bar.wait()
            return res
        return gather


def run_sharded(data, count, world, delta, prev, ops_for_rank, to_buf=lambda a: a, halo=S.HALO):
    data = np.asarray(data, np.uint8)
    L = data.size
    tg = ThreadGather(world)
    results = [None] * world
    errors = []

    def body(rank):
        try:
            lo, hi = S.local_range(L, world, rank, halo)
            results[rank] = S.sharded_decode(to_buf(data[lo:hi]), lo, L, count, delta, prev,
                                             ops_for_rank(rank), world=world, rank=rank,
                                             all_gather=tg.for_rank(rank))
        except BaseException as e:  # noqa: BLE001 - surfaced below
            errors.append(e)
            tg.bar.abort()

    th = [threading.Thread(target=body, args=(g,)) for g in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errors:
        raise errors[0]
    return results


def assemble(results, count):
    out = np.zeros(max(count, 0), np.uint32)
    glob = results[0][2]
    for off, vals, g in results:
        assert g == glob  # every rank reports the same whole-stream result
        v = vals.cpu().numpy().view(np.uint32) if hasattr(vals, "cpu") else np.asarray(vals, np.uint32)
        out[off:off + v.size] = v
    return glob, out


def check_against_whole(data, count, world, delta=True, prev=0, ops_for_rank=lambda g: OracleOps(),
                        to_buf=lambda a: a):
    res = run_sharded(data, count, world, delta, prev, ops_for_rank, to_buf)
    glob, out = assemble(res, count)
    if delta:
        want_r, want = oracle().decode_delta(np.asarray(data, np.uint8), count, prev, STRICT)
    else:
        want_r, want = oracle().decode(np.asarray(data, np.uint8), count, STRICT)
    assert glob == tuple(want_r), (glob, want_r)
    if want_r[0] == 0:
        np.testing.assert_array_equal(out[:count], want[:count])
    else:  # values before the error position are specified
        k = want_r[1]
        np.testing.assert_array_equal(out[:k], want[:k])
    return glob


# ------------------------------------------------------------------ host logic

def test_cuts_cover_and_align():
    for L in [0, 1, 15, 16, 17, 1000, 123457]:
        for w in [1, 2, 3, 8]:
            c = S.shard_cuts(L, w)
            assert c[0] == 0 and c[-1] == L and len(c) == w + 1
            assert all(a <= b for a, b in zip(c, c[1:]))
            assert all(x % 16 == 0 for x in c[1:-1])


def test_resync_lands_on_integer_starts():
    rng = np.random.default_rng(5)
    vals = W.mixed_values(20000, 5)
    enc = oracle().encode_sequence(vals)
    starts = set(np.concatenate([[0], np.cumsum([oracle().encoded_size(int(v)) for v in vals])]).tolist())
    for cut in range(0, enc.size, 13):
        pos, found = S.resync(enc, 0, cut, enc.size)
        assert found and pos in starts and pos >= cut and pos - cut <= 4


def test_combine_results_first_error_wins():
    recs = [(0, 5, 40, 0, 5), (2, 3, 17, 40, 9), (1, 0, 0, 90, 4)]
    assert S.combine_results(recs) == (2, 8, 57)
    assert S.combine_results([(0, 5, 40, 0, 5), (0, 0, 0, 40, 0)]) == (0, 5, 40)
    assert S.combine_results([(0, 0, 0, 0, 0)]) == (0, 0, 0)


# ------------------------------------------------ oracle-emulated W ranks (CPU)

def _gaps(n, seed, hi=1 << 20):
    rng = np.random.default_rng(seed)
    return rng.integers(0, hi, n, dtype=np.uint64).astype(np.uint32)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("delta", [False, True])
def test_sharded_equals_whole_stream(world, delta):
    gaps = W.mixed_values(30000, world)
    enc = oracle().encode_sequence(gaps)
    check_against_whole(enc, gaps.size, world, delta, prev=0xFFFFFF00)


@pytest.mark.parametrize("world", [2, 5])
def test_sharded_count_limits(world):
    gaps = _gaps(5000, 11)
    enc = oracle().encode_sequence(gaps)
    for count in [0, 1, 777, 2500, 4999, 5000, 5001, 9000]:
        check_against_whole(enc, count, world, True, prev=3)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_tiny_and_empty_streams(world):
    for n in [0, 1, 2, 3, 7, 40]:
        enc = oracle().encode_sequence(_gaps(n, n, 1 << 32))
        for count in {0, n, n + 1}:
            check_against_whole(enc, count, world, True, prev=1)


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_truncated_tail(world):
    enc = oracle().encode_sequence(_gaps(3000, 2, 1 << 32))
    for cut in [1, 2, 3, 4]:
        check_against_whole(enc[:-cut], 3000, world, True)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_malformed(world):
    base = oracle().encode_sequence(_gaps(4000, 3, 1 << 28))
    L = base.size
    for where in [0.1, 0.5, 0.74, 0.99]:
        p = int(L * where)
        # a non-canonical 5-byte integer (fifth byte >= 0x10) at an integer start
        bad = base.copy()
        q = S.resync(bad, 0, p, L)[0]
        fifth = np.array([0x81, 0x82, 0x83, 0x84, 0x7F], np.uint8)
        bad = np.concatenate([bad[:q], fifth, bad[q:]])
        check_against_whole(bad, 4001, world, True)
        # an over-long continuation run (longer than the resync halo) across a cut
        for runlen in [6, S.HALO + 3, 3 * S.HALO]:
            c = S.shard_cuts(L, world)[1]
            q = S.resync(base, 0, max(0, c - 7), L)[0]
            run = np.full(runlen, 0x85, np.uint8)
            bad = np.concatenate([base[:q], run, base[q:]])
            check_against_whole(bad, 4000, world, True)
            check_against_whole(bad, 4000, world, False)


# --------------------------------------------- real processes over gloo (CPU)

def _gloo_worker(rank, world, port, path, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        data = np.fromfile(path, np.uint8)
        count = int((data < 0x80).sum())
        lo, hi = S.local_range(data.size, world, rank)
        off, vals, glob = S.sharded_decode(data[lo:hi], lo, data.size, count, True, 7, OracleOps())
        q.put((rank, off, np.asarray(vals, np.uint32).tobytes(), glob))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_world2(tmp_path, world):
    import socket

    import torch.multiprocessing as mp

    gaps = W.mixed_values(50000, 9)
    enc = oracle().encode_sequence(gaps)
    path = str(tmp_path / "stream.bin")
    enc.tofile(path)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(g, world, port, path, q)) for g in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_r, want = oracle().decode_delta(enc, gaps.size, 7, STRICT)
    out = np.zeros(gaps.size, np.uint32)
    for rank, off, raw, glob in got:
        v = np.frombuffer(raw, np.uint32)
        out[off:off + v.size] = v
        assert glob == tuple(want_r)
    np.testing.assert_array_equal(out, want)


# ----------------------------------------------------------------------- GPU

def byte_weight_sum(seg) -> int:
    """The totals pass's sum of a byte range starting at an integer boundary:
    every byte's 7-bit digit times 128^(continuation bytes right before it in
    its integer), mod 2^32 -- the values of the integers ending in the range
    plus the partial value of an integer running past its end."""
    b = np.asarray(seg, np.int64)
    n = b.size
    if n == 0:
        return 0
    idx = np.arange(n)
    last = np.maximum.accumulate(np.where(b < 0x80, idx, -1))
    prev_term = np.concatenate([[-1], last[:-1]])
    run = idx - prev_term - 1
    w = np.where(run < 5, np.left_shift(1, 7 * np.minimum(run, 4)), 0)
    return int(((b & 0x7F) * w).sum() & 0xFFFFFFFF)


@pytest.mark.gpu
def test_totals_pass_matches_oracle(cuda):
    import torch

    ops = S.CudaShardOps(cuda)
    rng = np.random.default_rng(1)
    gaps = W.mixed_values(300000, 1)
    enc = oracle().encode_sequence(gaps)
    starts = np.concatenate([[0], np.cumsum([oracle().encoded_size(int(v)) for v in gaps[:2000]])])
    dev = torch.from_numpy(np.concatenate([np.zeros(64, np.uint8), enc])).to(cuda)
    for a in list(starts[:40]) + [int(starts[1999])]:
        for ln in [0, 1, 5, 16, 17, 100, 4095, 4096, 4097, 70000, enc.size - int(a)]:
            seg = enc[a:a + ln]
            n = int((seg < 0x80).sum())
            c, s = ops.totals(dev[64 + a:64 + a + seg.size])
            assert c == n
            assert s == byte_weight_sum(seg), (a, ln)
            if seg.size and seg[-1] < 0x80:  # ends at an integer boundary: the value sum
                _, vals = oracle().decode(seg, n, STRICT)
                assert s == int(vals.astype(np.uint64).sum() & 0xFFFFFFFF)
    # count is the terminator count on arbitrary bytes too
    junk = rng.integers(0, 256, 1 << 20, dtype=np.uint8)
    c, _ = ops.totals(torch.from_numpy(junk).to(cuda)[3:])
    assert c == int((junk[3:] < 0x80).sum())


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 3, 5])
def test_c_abi_sharded_over_virtual_gpus(cuda, n):
    """mvb_decode_delta_sharded: the whole stream's decode_delta_stream result
    and values from n shards (all on device 0), including count limits,
    truncation, malformed runs and prev wrap-around."""
    import ctypes

    import torch

    from paper_1503_07387_b200 import _lib

    L = _lib.lib()
    gaps = W.mixture(400000, 91, 0.3, (1, 127), (128, 70000))
    enc = oracle().encode_sequence(gaps)
    bad = enc.copy()
    bad[200001:200007] = 0x80  # a 7-byte run: malformed
    cases = [(enc, gaps.size, 7), (enc, 123457, 0), (enc[:-1], gaps.size, 0xFFFFFFF0), (bad, gaps.size, 3),
             (enc, gaps.size + 10, 5), (enc[:9], 5, 1)]
    for data, count, prev in cases:
        data = np.ascontiguousarray(data)
        cuts = np.zeros(n + 1, np.uint64)
        assert L.mvb_shard_cuts(data.ctypes.data, data.size, n, cuts.ctypes.data) == 0
        ins = [torch.from_numpy(data[int(cuts[g]):int(cuts[g + 1])].copy()).to(cuda) for g in range(n)]
        outs = [torch.full((max(x.numel(), 1),), -1, dtype=torch.int32, device=cuda) for x in ins]
        devs = (ctypes.c_int * n)(*([cuda.index or 0] * n))
        in_p = (ctypes.c_void_p * n)(*[x.data_ptr() if x.numel() else None for x in ins])
        lens = (ctypes.c_size_t * n)(*[x.numel() for x in ins])
        out_p = (ctypes.c_void_p * n)(*[o.data_ptr() for o in outs])
        offs = np.zeros(n, np.uint64)
        res = _lib.MvbResult()
        rc = L.mvb_decode_delta_sharded(n, devs, in_p, lens, count, prev, out_p, offs.ctypes.data, ctypes.byref(res))
        ro, oo = oracle().decode_delta(data, count, prev)
        assert rc == ro[0] and (res.status, res.values_written, res.bytes_consumed) == tuple(ro), (n, count, rc, ro)
        for g in range(n):
            a = int(offs[g])
            b = min(int(offs[g + 1]) if g + 1 < n else ro[1], ro[1])
            if b > a:
                got = outs[g][:b - a].cpu().numpy().view(np.uint32)
                assert np.array_equal(got, oo[a:b]), (n, count, g)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_cuda_equals_whole_stream(cuda, world):
    import torch

    gaps = W.mixed_values(1_000_000, world + 40)
    enc = oracle().encode_sequence(gaps)
    ops = [S.CudaShardOps(cuda) for _ in range(world)]

    def to_buf(a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(cuda)

    for delta in (False, True):
        check_against_whole(enc, gaps.size, world, delta, prev=11, ops_for_rank=lambda g: ops[g], to_buf=to_buf)
    # errors are reported exactly across shards too
    bad = enc.copy()
    q = S.resync(bad, 0, int(bad.size * 0.6), bad.size)[0]
    bad = np.concatenate([bad[:q], np.full(40, 0x90, np.uint8), bad[q:]])
    check_against_whole(bad, gaps.size, world, True, ops_for_rank=lambda g: ops[g], to_buf=to_buf)
    check_against_whole(enc[:-1], gaps.size, world, True, ops_for_rank=lambda g: ops[g], to_buf=to_buf)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_device_shards_equal_whole_stream(cuda, world):
    """DeviceShard phases (pre-pass -> record exchange -> carry -> decode) for W
    virtual shards on one GPU; the exchange is a device copy standing in for
    the NCCL all-gather."""
    import torch

    gaps = W.mixed_values(2_000_000, world + 70)
    for data in (oracle().encode_sequence(gaps), None):
        if data is None:  # malformed: an over-long run in the middle
            enc = oracle().encode_sequence(gaps)
            q = S.resync(enc, 0, enc.size // 2 + 5, enc.size)[0]
            data = np.concatenate([enc[:q], np.full(30, 0x88, np.uint8), enc[q:]])
        L = data.size
        n_ints = int((data < 0x80).sum())
        for delta in (False, True):
            shards = []
            for g in range(world):
                lo, hi = S.local_range(L, world, g)
                shards.append(S.DeviceShard(torch.from_numpy(data[lo:hi].copy()).to(cuda), lo, L, delta,
                                            prev=0xFFFFFFF0, world=world, rank=g))
            recs_all = torch.zeros(world * 2, dtype=torch.int64, device=cuda)
            for sh in shards:
                sh.prepass()
            for g, sh in enumerate(shards):
                recs_all[2 * g:2 * g + 2] = sh.rec
            for sh in shards:
                sh.recs.copy_(recs_all)
                sh.decode()
            torch.cuda.synchronize()
            locs = [sh.local_result() for sh in shards]
            got = np.zeros(n_ints, np.uint32)
            off = 0
            for sh, lr in zip(shards, locs):
                v = sh.out[:lr[1]].cpu().numpy().view(np.uint32)
                got[off:off + v.size] = v
                off += v.size
            glob = S.combine_results(locs)
            if delta:
                want_r, want = oracle().decode_delta(data, n_ints, 0xFFFFFFF0, STRICT)
            else:
                want_r, want = oracle().decode(data, n_ints, STRICT)
            assert glob == tuple(want_r), (world, delta, glob, want_r)
            k = want_r[1]
            np.testing.assert_array_equal(got[:k], want[:k])


@pytest.mark.gpu
def test_cpp_driver_sharded_c_abi():
    """The C++ caller of mvb_decode_delta_sharded (tests/cpp/sharded_abi_test.cpp):
    1, 2, 3, 5 and 8 shards on this process's GPUs (repeated when there is one)
    against the oracle -- plain, count-limited, truncated and malformed streams."""
    import subprocess

    from paper_1503_07387_b200 import build as B

    exe = B.build_cpp_tests(verbose=False)
    r = subprocess.run([exe, "400000", "1", "2", "3", "5", "8"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "25/25 sharded C-ABI cases passed" in r.stdout, r.stdout
