"""ListFile ingestion: the reference's on-disk list
container read into device batch descriptors for the batched decode.

Format (/root/reference/proj/core/include/mvb/list_file.hpp:13-16), all
little-endian: magic "MVB1" | flags u32 (bit 0 = delta-coded) | count u32 |
payload_len u32, then payload_len payload bytes.  ``read_list`` /
``write_list`` mirror list_file.cpp:44-87 (same errors: bad magic, truncated
header or payload, and with ``validate_payload`` a payload that is not
exactly ``count`` canonical integers spanning exactly ``payload_len`` bytes,
list_file.cpp:25-42).  ``read_batch`` gathers every container of one or more
files (containers may sit back to back in a file) into one concatenated
payload with per-list byte and integer offsets; ``decode_batch`` decodes the
whole batch on the GPU in one launch per coding kind
(``mvb_decode[_delta]_lists_device``), each list from prev 0 exactly as the
reference runner's per-list decode (tools/bench/runner.cpp:28-61).
"""
from __future__ import annotations

import io
import os
import struct
from dataclasses import dataclass
from typing import Optional, Iterable, List, Sequence, Union

import numpy as np

from .mvb import EncodedBuffer

MAGIC = b"MVB1"
HEADER_BYTES = 16
MAX_ENCODED_BYTES = 5


class ListFileError(RuntimeError):
    """list_file.hpp:18-20"""


def payload_is_canonical(payload: np.ndarray, count: int) -> bool:
    """list_file.cpp:25-42, vectorised: exactly `count` integers of 1..5
    bytes, minimal length (no trailing 0x00 after a continuation byte), fifth
    byte below 0x10, covering the whole payload."""
    b = np.asarray(payload, np.uint8)
    if count == 0:
        return b.size == 0
    if b.size == 0 or b[-1] >= 0x80:
        return False  # truncated last integer (or extra bytes without an end)
    ends = np.flatnonzero(b < 0x80)
    if ends.size != count:
        return False
    lens = np.diff(np.concatenate([[-1], ends]))
    if (lens > MAX_ENCODED_BYTES).any():
        return False
    last = b[ends]
    if ((lens == MAX_ENCODED_BYTES) & (last >= 0x10)).any():
        return False
    if ((lens > 1) & (last == 0)).any():
        return False  # non-minimal
    return True


def write_list(sink, buf: EncodedBuffer, delta_coded: Optional[bool] = None) -> int:
    """list_file.cpp:44-55: header + payload; returns the bytes written.  The
    flag is the buffer's own delta_coded (list_file.cpp:50) unless given."""
    if delta_coded is None:
        delta_coded = bool(buf.delta_coded)
    payload = np.ascontiguousarray(buf.bytes, np.uint8)
    if payload.size > 0xFFFFFFFF:
        raise ListFileError("write_list: payload exceeds 32-bit length")
    sink.write(MAGIC + struct.pack("<III", 1 if delta_coded else 0, int(buf.count), payload.size))
    sink.write(payload.tobytes())
    return HEADER_BYTES + payload.size


def write_list_file(path, buf: EncodedBuffer, delta_coded: Optional[bool] = None) -> int:
    with open(path, "wb") as f:
        return write_list(f, buf, delta_coded)


@dataclass
class ListRecord:
    buf: EncodedBuffer
    delta_coded: bool


def read_list(source, validate_payload: bool = True) -> ListRecord:
    """list_file.cpp:63-87."""
    magic = source.read(4)
    if len(magic) != 4 or magic != MAGIC:
        raise ListFileError("read_list: bad magic")
    hdr = source.read(12)
    if len(hdr) != 12:
        raise ListFileError("read_list: truncated header")
    flags, count, payload_len = struct.unpack("<III", hdr)
    payload = source.read(payload_len)
    if len(payload) != payload_len:
        raise ListFileError("read_list: truncated payload")
    b = np.frombuffer(payload, np.uint8)
    if validate_payload and not payload_is_canonical(b, count):
        raise ListFileError(f"read_list: payload is not {count} canonical integers")
    return ListRecord(EncodedBuffer(b, count, (flags & 1) != 0), (flags & 1) != 0)


def read_list_file(path, validate_payload: bool = True) -> ListRecord:
    with open(path, "rb") as f:
        return read_list(f, validate_payload)


@dataclass
class ListBatch:
    """Lists concatenated for one batched decode."""
    payload: np.ndarray       # uint8, all payloads back to back
    byte_offsets: np.ndarray  # uint64 [n + 1]
    int_offsets: np.ndarray   # uint64 [n + 1]
    delta: np.ndarray         # bool [n]

    @property
    def n_lists(self) -> int:
        return int(self.delta.size)


def read_batch(paths: Union[str, os.PathLike, Sequence], validate_payload: bool = True) -> ListBatch:
    """Every ListFile container of the given file(s), in order."""
    if isinstance(paths, (str, os.PathLike)):
        paths = [paths]
    recs: List[ListRecord] = []
    for p in paths:
        with open(p, "rb") as f:
            data = f.read()
        src = io.BytesIO(data)
        while src.tell() < len(data):
            recs.append(read_list(src, validate_payload))
    return batch_of(recs)


def batch_of(recs: Iterable[ListRecord]) -> ListBatch:
    recs = list(recs)
    sizes = np.array([r.buf.bytes.size for r in recs], np.uint64)
    counts = np.array([r.buf.count for r in recs], np.uint64)
    bo = np.zeros(len(recs) + 1, np.uint64)
    io_ = np.zeros(len(recs) + 1, np.uint64)
    np.cumsum(sizes, out=bo[1:])
    np.cumsum(counts, out=io_[1:])
    payload = (np.concatenate([np.asarray(r.buf.bytes, np.uint8) for r in recs]) if recs
               else np.zeros(0, np.uint8))
    return ListBatch(payload, bo, io_, np.array([r.delta_coded for r in recs], bool))


def decode_batch(batch: ListBatch, device=None):
    """Decode every list of the batch on the GPU: one launch per coding kind
    (delta lists, plain lists), longest lists first.  Returns (values: uint32
    numpy array in list order, results: int64 numpy array [n, 3] = per-list
    (status, values_written, bytes_consumed))."""
    import torch

    from .mvb import Decoder

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    n = batch.n_lists
    total = int(batch.int_offsets[-1]) if n else 0
    values = np.zeros(total, np.uint32)
    results = np.zeros((n, 3), np.int64)
    d = Decoder(dev, 1 << 12)
    for kind in (True, False):
        sel = np.flatnonzero(batch.delta == kind)
        if sel.size == 0:
            continue
        # this kind's lists as their own contiguous batch (host-side gather)
        spans = [batch.payload[int(batch.byte_offsets[l]):int(batch.byte_offsets[l + 1])] for l in sel]
        counts = (batch.int_offsets[sel + 1] - batch.int_offsets[sel]).astype(np.uint64)
        bo = np.zeros(sel.size + 1, np.uint64)
        io_ = np.zeros(sel.size + 1, np.uint64)
        np.cumsum([x.size for x in spans], out=bo[1:])
        np.cumsum(counts, out=io_[1:])
        src = torch.from_numpy(np.concatenate(spans) if spans else np.zeros(0, np.uint8)).to(dev)
        out = torch.zeros(max(int(io_[-1]), 1), dtype=torch.int32, device=dev)
        res = torch.zeros(sel.size * 3, dtype=torch.int64, device=dev)
        order = np.argsort(-np.diff(bo.astype(np.int64)), kind="stable").astype(np.uint32)
        d.decode_lists(src, torch.from_numpy(bo.view(np.int64)).to(dev), torch.from_numpy(io_.view(np.int64)).to(dev),
                       out, order=torch.from_numpy(order.view(np.int32)).to(dev), results=res, delta=kind)
        o = out.cpu().numpy().view(np.uint32)
        r = res.cpu().numpy().reshape(-1, 3)
        for k, l in enumerate(sel):
            a, b = int(io_[k]), int(io_[k + 1])
            values[int(batch.int_offsets[l]):int(batch.int_offsets[l]) + (b - a)] = o[a:b]
            results[l] = r[k]
    return values, results
