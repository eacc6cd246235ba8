"""Byte-range sharded decode of one VByte stream across the GPUs of a node
(BASELINE.json config 4).

The stream of L bytes is cut into `world` byte ranges at 16-byte-aligned cuts.
Rank g holds bytes [lo_g, hi_g) = its range plus a small halo on both sides.
Each rank

1. resynchronises: its shard starts at the first integer start at or after
   its cut (the first byte whose predecessor terminates an integer; in
   canonical data at most 4 bytes after the cut) and ends where the next
   rank's shard starts -- every integer is owned by exactly one shard;
2. runs the totals pass over its shard (delta decode, every rank but the
   last): integer count and the sum of its gaps mod 2^32, one read of the
   shard (``mvb_delta_totals_device``, last unit first so that the decode
   pass finds the shard's head in L2);
3. exchanges one small record per rank (start, end, count, sum) with a
   single all-gather -- the only collective; the bulk data never moves;
4. decodes its shard as a standalone stream with ``count`` = its integers and
   ``prev`` = the caller's prev plus the gap sums of all earlier shards, into
   its local output (global offset = integers in earlier shards): ranks that
   ran the totals pass decode with it (``mvb_decode_delta_totaled_device``),
   the last rank in one pass (totals and decode interleaved).

The per-rank result is the reference's DecodeResult for the shard; the global
result is assembled by ``combine_results`` exactly as decode_delta_scalar
(/root/reference/proj/core/src/vbyte.cpp:63-74) would report on the whole
stream: the first shard that is not OK decides, with its progress counters
offset by the earlier shards' totals.

The device work is behind a small ``ShardOps`` interface: ``CudaShardOps``
runs the sm_100a kernels through the C ABI; tests substitute a CPU oracle to
check the host logic under a multi-process ``gloo`` group (only one GPU is
available to the test environment).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

HALO = 16  # >= 5 bytes: enough to find the integer boundary after a cut in canonical data


def shard_cuts(total_len: int, world: int, align: int = 16) -> List[int]:
    """Byte cuts c_0 = 0 <= c_1 <= ... <= c_world = total_len (interior cuts aligned)."""
    cuts = [0]
    for g in range(1, world):
        c = (total_len * g // world) // align * align
        cuts.append(max(cuts[-1], c))
    cuts.append(total_len)
    return cuts


def local_range(total_len: int, world: int, rank: int, halo: int = HALO) -> Tuple[int, int]:
    """Bytes [lo, hi) rank `rank` must hold: its range plus halos."""
    cuts = shard_cuts(total_len, world)
    return max(0, cuts[rank] - halo), min(total_len, cuts[rank + 1] + halo)


def resync(buf: np.ndarray, buf_lo: int, cut: int, total_len: int, halo: int = HALO) -> Tuple[int, bool]:
    """First integer start at or after `cut` (stream coordinates): the byte
    after the first terminator (high bit clear) in the window
    [cut-1, cut+halo-1).  Both neighbouring ranks hold that window, so they
    reach the same decision.  Returns (position, found); when the window has
    no terminator the data is not canonical (a continuation run longer than
    `halo`) and the position is the window end -- see sharded_decode for how
    the error is still reported exactly."""
    if cut <= 0:
        return 0, True
    if cut >= total_len:
        return total_len, True
    rel = cut - 1 - buf_lo
    stop = min(total_len, cut + halo - 1) - buf_lo
    if rel < 0 or stop > len(buf):
        raise ValueError("buffer does not cover the resync window of the cut")
    hits = np.flatnonzero(np.asarray(buf[rel:stop], dtype=np.uint8) < 0x80)
    if hits.size == 0:
        return buf_lo + stop, False
    return cut + int(hits[0]), True


def list_ranges(byte_off: Sequence[int], world: int) -> List[int]:
    """Cut a batch of independent lists (BASELINE.json config 3) into `world`
    contiguous list ranges balanced by compressed bytes (the
    lists are independent units, so no exchange is needed).  Returns
    world + 1 list indices; rank r decodes lists [cuts[r], cuts[r+1]), whose
    output offsets are int_off[cuts[r]] ... in the whole batch's output."""
    bo = np.asarray(byte_off, dtype=np.int64)
    n = bo.size - 1
    if world < 1:
        raise ValueError("world must be >= 1")
    total = int(bo[-1] - bo[0])
    targets = [int(bo[0]) + (total * r) // world for r in range(world + 1)]
    cuts = [int(np.searchsorted(bo[:n + 1], t, side="left")) for t in targets]
    cuts[0], cuts[-1] = 0, n
    for r in range(1, world + 1):  # monotone even for empty ranges
        cuts[r] = max(cuts[r], cuts[r - 1])
    return cuts


@dataclass
class ShardPlan:
    rank: int
    world: int
    start: int       # stream position of the shard's first byte
    end: int         # stream position after the shard's last byte
    end_synced: bool  # the end window held a terminator


def plan_shard(buf: np.ndarray, buf_lo: int, total_len: int, world: int, rank: int) -> ShardPlan:
    cuts = shard_cuts(total_len, world)
    start, _ = resync(buf, buf_lo, cuts[rank], total_len)
    if rank == world - 1:
        end, synced = total_len, True
    else:
        end, synced = resync(buf, buf_lo, cuts[rank + 1], total_len)
    return ShardPlan(rank, world, start, max(start, end), synced)


def shard_counts(recs: Sequence[Sequence[int]], count: int) -> List[int]:
    """Integers each shard decodes, given the gathered (start, end, n, sum,
    end_synced) records and the caller's global count.  Every shard but the
    last decodes its own integers, capped by what is left of `count`; a shard
    whose end window had no terminator asks for one more, so that its decode
    runs into the over-long continuation run and reports it exactly as the
    whole-stream decode would.  The last shard is asked for all that is
    left, so a short stream reports `truncated` as decode_scalar does
    (vbyte.cpp:47-57)."""
    out, left = [], count
    for g, r in enumerate(recs):
        want = left if g == len(recs) - 1 else min(left, r[2] + (0 if r[4] else 1))
        want = max(0, want)
        out.append(want)
        left -= want
    return out


def combine_results(records: Sequence[Sequence[int]]) -> Tuple[int, int, int]:
    """Global DecodeResult from per-shard (status, values_written,
    bytes_consumed, shard_start, integers_requested) records in rank order:
    the first shard that is not OK decides; otherwise bytes_consumed is the
    end of the last shard that decoded anything."""
    written = consumed = 0
    for status, vw, bc, start, k in records:
        if status != 0:
            return int(status), written + int(vw), int(start) + int(bc)
        written += int(vw)
        if k > 0:
            consumed = int(start) + int(bc)
    return 0, written, consumed


class ShardOps:
    """Device operations a shard needs (totals pre-pass, decode)."""

    def totals(self, shard) -> Tuple[int, int]:  # (integers, gap sum mod 2^32)
        raise NotImplementedError

    def decode(self, shard, count: int, prev: int, delta: bool, out=None):
        raise NotImplementedError  # -> ((status, written, consumed), values)


class CudaShardOps(ShardOps):
    """sm_100a kernels through the C ABI (torch CUDA tensors)."""

    def __init__(self, device):
        import torch

        from . import _lib, mvb

        self.torch = torch
        self.device = torch.device(device)
        self.lib = _lib.lib()
        self.dec = mvb.Decoder(self.device)
        self.rec = torch.zeros(2, dtype=torch.int64, device=self.device)  # [count, gap sum]

    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def totals_async(self, shard):
        """Queue the totals pass; returns the device record [count, gap sum] without syncing."""
        n = shard.numel()
        self.dec._ensure(max(n, 1))
        rc = self.lib.mvb_delta_totals_device(shard.data_ptr() if n else None, n, self.rec.data_ptr(),
                                              self.dec.ws.data_ptr(), self.dec.ws_bytes, self._stream())
        if rc != 0:
            raise RuntimeError(f"mvb_delta_totals_device failed ({rc})")
        return self.rec

    def totals(self, shard) -> Tuple[int, int]:
        r = self.totals_async(shard).cpu().tolist()
        return int(r[0]), int(r[1]) & 0xFFFFFFFF

    def decode(self, shard, count: int, prev: int, delta: bool, out=None):
        torch = self.torch
        if out is None:
            out = torch.empty(max(count, 1), dtype=torch.int32, device=self.device)
        if delta:
            self.dec.decode_delta(shard, count, prev, out, 0, in_len=shard.numel())
        else:
            self.dec.decode(shard, count, out, 0, in_len=shard.numel())
        r = self.dec.result()
        return (int(r.status), r.values_written, r.bytes_consumed), out[:count]


def _all_gather_records(record: List[int], group=None) -> List[List[int]]:
    """One int64 record per rank (the only collective of the sharded decode)."""
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor(record, dtype=torch.int64, device=dev)
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, t, group=group)
    return [p.cpu().tolist() for p in parts]


def _window_view(buf, buf_lo: int, total_len: int, cuts: Sequence[int], rank: int) -> np.ndarray:
    """Host copy of just the bytes resync reads (device buffers: 2 x HALO bytes)."""
    if not hasattr(buf, "cpu"):
        return np.asarray(buf, np.uint8)
    host = np.zeros(len(buf), np.uint8)  # placeholder bytes are never inspected
    for c in (cuts[rank], cuts[rank + 1]):
        a, b = max(0, c - 1 - buf_lo), min(len(buf), c + HALO - 1 - buf_lo)
        if b > a:
            host[a:b] = buf[a:b].cpu().numpy()
    return host


def sharded_decode(buf, buf_lo: int, total_len: int, count: int, delta: bool, prev: int,
                   ops: ShardOps, world: Optional[int] = None, rank: Optional[int] = None,
                   group=None, all_gather=None, out=None):
    """Decode this rank's shard of a stream distributed by byte range (strict
    mode; the sharded path serves canonical posting data, BASELINE config 4).

    ``buf`` holds stream bytes [buf_lo, buf_lo + len(buf)) -- at least
    ``local_range(total_len, world, rank)`` -- as a numpy array or a CUDA
    tensor; ``count`` and ``prev`` are the whole-stream decode arguments.
    Returns (global_offset, values, global_result): this rank's values are
    out[global_offset : global_offset + len(values)] of the whole-stream
    decode, and global_result is the whole-stream DecodeResult (identical on
    every rank).
    """
    import torch.distributed as dist

    if world is None:
        world = dist.get_world_size(group)
    if rank is None:
        rank = dist.get_rank(group)
    cuts = shard_cuts(total_len, world)
    plan = plan_shard(_window_view(buf, buf_lo, total_len, cuts, rank), buf_lo, total_len, world, rank)
    shard = buf[plan.start - buf_lo: plan.end - buf_lo]
    n, s = ops.totals(shard)
    gather = all_gather or (lambda r: _all_gather_records(r, group))
    recs = gather([plan.start, plan.end, n, s if delta else 0, int(plan.end_synced)])
    want = shard_counts(recs, count)
    offset = sum(want[:rank])
    carry = (prev + sum(r[3] for r in recs[:rank])) & 0xFFFFFFFF
    local, values = ops.decode(shard, want[rank], carry if delta else 0, delta, out)
    status_recs = gather([local[0], local[1], local[2], plan.start, want[rank]])
    return offset, values, combine_results(status_recs)


class DeviceShard:
    """One rank's shard, decoded with no host round trip (bench / device-resident path).

    Every pass queues, on the current stream: the totals pre-pass (delta, all
    ranks but the last -- nobody needs the last shard's sum), an all-gather of
    a 16-byte record {count, gap sum} per rank, the carry kernel, and the
    decode with its starting value read from device memory.  Plain decode
    needs no exchange at all: each shard decodes independently and only the
    output offsets (metadata, ``result()``) use the gathered counts.

    The shard is decoded with ``count`` = its byte length (an upper bound on
    its integers), i.e. "every integer in the stream": a shard that ends
    cleanly reports truncated with all bytes consumed, which ``result()``
    reads as OK -- the whole-stream decode with count = number of integers.
    """

    RECORD_WORDS = 2

    def __init__(self, buf, buf_lo: int, total_len: int, delta: bool, prev: int = 0,
                 world: int = 1, rank: int = 0, group=None, gather=None):
        import torch

        from . import _lib, mvb

        self.torch = torch
        self.lib = _lib.lib()
        self.device = buf.device
        self.delta, self.prev = delta, prev & 0xFFFFFFFF
        self.world, self.rank, self.group = world, rank, group
        self.total_len = total_len
        cuts = shard_cuts(total_len, world)
        self.plan = plan_shard(_window_view(buf, buf_lo, total_len, cuts, rank), buf_lo, total_len, world, rank)
        self.shard = buf[self.plan.start - buf_lo: self.plan.end - buf_lo]
        self.bound = int(self.shard.numel())
        self.out = torch.empty(max(self.bound, 1), dtype=torch.int32, device=self.device)
        self.rec = torch.zeros(self.RECORD_WORDS, dtype=torch.int64, device=self.device)
        self.recs = torch.zeros(world * self.RECORD_WORDS, dtype=torch.int64, device=self.device)
        self.carry = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.dec = mvb.Decoder(self.device, capacity_bytes=max(self.bound, 1))
        self.gather = gather
        self.launches_per_pass = _lib.kernels_per_decode(0) + (2 if delta and world > 1 and rank < world - 1 else
                                                             1 if delta and world > 1 else 0)

    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def prepass(self):
        """Totals of this shard into the local record (delta, not the last rank):
        one read of the shard, last unit first; the workspace keeps the per-unit
        totals for decode()."""
        if not self.delta or self.world == 1 or self.rank == self.world - 1:
            return
        n = self.bound
        self.dec._ensure(max(n, 1))
        rc = self.lib.mvb_delta_totals_device(self.shard.data_ptr() if n else None, n, self.rec.data_ptr(),
                                              self.dec.ws.data_ptr(), self.dec.ws_bytes, self._stream())
        if rc != 0:
            raise RuntimeError(f"mvb_delta_totals_device failed ({rc})")

    def exchange(self):
        """All-gather of the records (the only collective)."""
        if self.gather is not None:
            self.gather(self.recs, self.rec)
        else:
            import torch.distributed as dist

            dist.all_gather_into_tensor(self.recs, self.rec, group=self.group)

    def decode(self):
        n, s = self.bound, self._stream()
        self.dec._ensure(max(n, 1))
        ws, wsb = self.dec.ws.data_ptr(), self.dec.ws_bytes
        if self.delta and self.world > 1:
            rc = self.lib.mvb_shard_carry_device(self.recs.data_ptr(), self.world, self.rank, self.RECORD_WORDS,
                                                 self.prev, self.carry.data_ptr(), None, s)
            if rc != 0:
                raise RuntimeError(f"mvb_shard_carry_device failed ({rc})")
            if self.rank < self.world - 1:  # after this pass's totals pass (prepass)
                rc = self.lib.mvb_decode_delta_totaled_device(self.shard.data_ptr() if n else None, n, n, 0,
                                                              self.carry.data_ptr(),
                                                              self.out.data_ptr() if n else None,
                                                              self.dec.res.data_ptr(), ws, wsb, s)
            else:
                rc = self.lib.mvb_decode_delta_device_dprev(self.shard.data_ptr() if n else None, n, n,
                                                            self.carry.data_ptr(),
                                                            self.out.data_ptr() if n else None,
                                                            0, self.dec.res.data_ptr(), ws, wsb, s)
        elif self.delta:
            rc = self.lib.mvb_decode_delta_device(self.shard.data_ptr() if n else None, n, n, self.prev,
                                                  self.out.data_ptr() if n else None, 0, self.dec.res.data_ptr(),
                                                  ws, wsb, s)
        else:
            rc = self.lib.mvb_decode_device(self.shard.data_ptr() if n else None, n, n,
                                            self.out.data_ptr() if n else None, 0, self.dec.res.data_ptr(),
                                            ws, wsb, s)
        if rc != 0:
            raise RuntimeError(f"shard decode failed ({rc})")

    def run(self):
        """One pass over the shard (queued on the current stream).  NVTX ranges
         mark the three phases for timeline tools."""
        nvtx = self.torch.cuda.nvtx
        nvtx.range_push("mvb.shard.totals")
        self.prepass()
        nvtx.range_pop()
        if self.delta and self.world > 1:
            nvtx.range_push("mvb.shard.exchange")
            self.exchange()
            nvtx.range_pop()
        nvtx.range_push("mvb.shard.decode")
        self.decode()
        nvtx.range_pop()

    def local_result(self) -> List[int]:
        """(status, written, consumed, start, requested) with a clean end read as OK."""
        r = self.dec.result()
        status = int(r.status)
        if status == 1 and r.bytes_consumed == self.bound:
            status = 0
        return [status, int(r.values_written), int(r.bytes_consumed), self.plan.start, self.bound]

    def result(self, gather_records=None):
        """(global_offset, values, whole-stream DecodeResult); synchronises."""
        gather = gather_records or (lambda rec: _all_gather_records(rec, self.group))
        recs = gather(self.local_result()) if self.world > 1 else [self.local_result()]
        offset = sum(r[1] for r in recs[:self.rank])
        mine = recs[self.rank]
        return offset, self.out[:mine[1]], combine_results(recs)
