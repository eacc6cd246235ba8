"""Python mirror of the reference codec interface, backed by the CUDA C ABI.

Names, argument meaning and error behaviour follow the reference library
``mvbyte`` (paths relative to /root/reference/proj):

====================================  =========================================
this module                           reference
====================================  =========================================
DecodeMode / DecodeStatus             core/include/mvb/vbyte.hpp:38-43
DecodeResult                          core/include/mvb/vbyte.hpp:45-49
DecodeOptions                         core/include/mvb/decode.hpp:20-28
EncodedBuffer                         core/include/mvb/vbyte.hpp:26-30
encoded_size / encode_one             core/src/vbyte.cpp:9-31
encode_sequence / encode_deltas       core/src/vbyte.cpp:33-45
delta_encode / prefix_sum_scalar      core/src/vbyte.cpp:76-99
decode_stream / decode_scalar         core/src/decode.cpp:73-86, vbyte.cpp:47-61
decode_delta_stream / _delta_scalar   core/src/decode.cpp:88-102, vbyte.cpp:63-74
====================================  =========================================

Every decode runs the sm_100a kernel: host arrays (numpy / bytes) go through
the synchronous host drop-in (H2D copy, decode, D2H copy); torch CUDA tensors
go through the device entry points on the current stream.  ``decode_scalar``
and ``decode_stream`` are the same GPU decode because the reference defines
them to have identical results (decode.hpp:42-43).  ``DecodeOptions.path``
and ``scalar_handoff`` select CPU backends in the reference; they are accepted
for signature compatibility and do not change the result (the reference pins
that invariance, decode_test.cpp:333-362).
"""
from __future__ import annotations

import ctypes
import weakref
import enum
from dataclasses import dataclass, field
from typing import Optional, Union

import numpy as np

from . import _lib


class DecodeMode(enum.IntEnum):
    strict = 0      # reject integers whose fifth byte is >= 0x10
    permissive = 1  # take the fifth byte whole; value reduced mod 2^32


class DecodeStatus(enum.IntEnum):
    ok = 0
    truncated = 1
    malformed = 2


class DecodePath(enum.IntEnum):
    auto_select = 0
    portable = 1
    vector = 2


@dataclass
class DecodeResult:
    status: DecodeStatus = DecodeStatus.ok
    values_written: int = 0
    bytes_consumed: int = 0


@dataclass
class DecodeOptions:
    path: DecodePath = DecodePath.auto_select
    mode: DecodeMode = DecodeMode.strict
    scalar_handoff: int = 16


@dataclass
class EncodedBuffer:
    bytes: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    count: int = 0
    delta_coded: bool = False


class MvbError(RuntimeError):
    """A negative return code of the C ABI (API misuse or CUDA failure)."""


_ERRORS = {-1: "invalid argument", -2: "workspace too small", -3: "CUDA error", -4: "input decreases"}


def _check(rc: int) -> int:
    if rc < 0:
        raise MvbError(f"mvb_cuda: {_ERRORS.get(rc, rc)} ({rc})")
    return rc


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


def _u8(a) -> np.ndarray:
    if isinstance(a, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(a), dtype=np.uint8)
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint8))


def _ptr(a: np.ndarray) -> Optional[int]:
    return a.ctypes.data if a.size else None


# ------------------------------------------------------------------ encoder

def encoded_size(x: int) -> int:
    return int(_lib.lib().mvb_encoded_size(int(x) & 0xFFFFFFFF))


def encode_one(x: int) -> bytes:
    buf = (ctypes.c_uint8 * 5)()
    n = _lib.lib().mvb_encode_one(int(x) & 0xFFFFFFFF, buf)
    return bytes(buf[:n])


def encode_sequence(values) -> EncodedBuffer:
    v = _u32(values)
    L = _lib.lib()
    n = L.mvb_encoded_length(_ptr(v), v.size)
    out = np.empty(n, np.uint8)
    L.mvb_encode_sequence(_ptr(v), v.size, _ptr(out))
    return EncodedBuffer(out, int(v.size), False)


def encode_deltas(sorted_values) -> EncodedBuffer:
    """delta_encode + encode_sequence; raises ValueError (std::invalid_argument
    in the reference, vbyte.cpp:80-81) if the input decreases."""
    v = _u32(sorted_values)
    out = np.empty(5 * v.size, np.uint8)
    n = ctypes.c_size_t(0)
    bad = ctypes.c_size_t(0)
    rc = _lib.lib().mvb_encode_deltas(_ptr(v), v.size, _ptr(out), ctypes.byref(n), ctypes.byref(bad))
    if rc == -4:
        raise ValueError(f"delta_encode: input decreases at index {bad.value}")
    _check(rc)
    return EncodedBuffer(out[: n.value].copy(), int(v.size), True)


def delta_encode(values) -> np.ndarray:
    v = _u32(values).astype(np.int64)
    if v.size and np.any(np.diff(v) < 0):
        i = int(np.argmax(np.diff(v) < 0)) + 1
        raise ValueError(f"delta_encode: input decreases at index {i}")
    return np.diff(v, prepend=0).astype(np.uint32)


def prefix_sum_scalar(gaps, prev: int = 0) -> np.ndarray:
    g = _u32(gaps).astype(np.uint64)
    return ((np.cumsum(g, dtype=np.uint64) + np.uint64(prev)) & np.uint64(0xFFFFFFFF)).astype(np.uint32)


# ------------------------------------------------------------------ decode

def _is_cuda_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


def _mode_of(options) -> int:
    if options is None:
        return int(DecodeMode.strict)
    if isinstance(options, DecodeOptions):
        return int(options.mode)
    return int(DecodeMode(options))


def _check_in_tensor(inp, n: int) -> None:
    """A device input must be a contiguous uint8 CUDA tensor with >= n bytes."""
    torch = inp.__class__.__module__.startswith("torch") and __import__("torch")
    if not torch or not inp.is_cuda or inp.dtype != torch.uint8 or not inp.is_contiguous():
        raise MvbError("device input must be a contiguous uint8 CUDA tensor")
    if inp.numel() < n:
        raise MvbError("device input holds fewer than in_len bytes")


def _check_out_tensor(out, count: int, device) -> None:
    """A device output must be a contiguous int32/uint32 CUDA tensor on the
    input's device with >= count elements: the kernels write count*4
    contiguous bytes from out.data_ptr()."""
    if count == 0:
        return
    import torch

    if out is None or not isinstance(out, torch.Tensor) or not out.is_cuda:
        raise MvbError("decode on CUDA tensors needs a CUDA output tensor")
    if out.dtype not in (torch.int32, torch.uint32) or not out.is_contiguous():
        raise MvbError("device output must be a contiguous int32/uint32 tensor")
    if out.device != device:
        raise MvbError("device output must be on the input's device")
    if out.numel() < count:
        raise MvbError("device output holds fewer than count elements")


class Decoder:
    """Device-side decoder state: a workspace and a result slot on one GPU.

    ``decode(in, count, out)`` / ``decode_delta(in, count, prev, out)`` take
    torch CUDA tensors (uint8 input, int32/uint32 output), queue the kernel on
    the current stream and return immediately; ``result()`` syncs and reads the
    DecodeResult.  One Decoder must not be used by two streams at once."""

    def __init__(self, device=None, capacity_bytes: int = 1 << 20):
        import torch

        self.torch = torch
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.res = torch.zeros(3, dtype=torch.int64, device=self.device)  # 24-byte mvb_result
        self.ws = None
        self.ws_bytes = 0
        self._lists_ok = []  # validated (offset tensors (weak), versions, total integer count), newest last
        self._ensure(capacity_bytes)

    def _ensure(self, in_len: int):
        need = int(_lib.lib().mvb_workspace_bytes(int(in_len)))
        if need > self.ws_bytes:
            self.ws = self.torch.zeros(need, dtype=self.torch.uint8, device=self.device)
            self.ws_bytes = need

    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def decode(self, inp, count: int, out, mode: int = 0, in_len: Optional[int] = None) -> None:
        n = inp.numel() if in_len is None else int(in_len)
        _check_in_tensor(inp, n)
        _check_out_tensor(out, int(count), inp.device)
        self._ensure(n)
        _check(_lib.lib().mvb_decode_device(
            inp.data_ptr() if n else None, n, int(count), out.data_ptr() if count else None, int(mode),
            self.res.data_ptr(), self.ws.data_ptr(), self.ws_bytes, self._stream()))

    def decode_delta(self, inp, count: int, prev: int, out, mode: int = 0, in_len: Optional[int] = None) -> None:
        n = inp.numel() if in_len is None else int(in_len)
        _check_in_tensor(inp, n)
        _check_out_tensor(out, int(count), inp.device)
        self._ensure(n)
        _check(_lib.lib().mvb_decode_delta_device(
            inp.data_ptr() if n else None, n, int(count), int(prev) & 0xFFFFFFFF,
            out.data_ptr() if count else None, int(mode),
            self.res.data_ptr(), self.ws.data_ptr(), self.ws_bytes, self._stream()))

    def decode_lists(self, inp, byte_offsets, int_offsets, out, prev=None, order=None, results=None,
                     delta: bool = True, mode: int = 0) -> None:
        """Batched posting lists (mvb_decode[_delta]_lists_device): list l is
        inp[byte_offsets[l]:byte_offsets[l+1]] with int_offsets[l+1] -
        int_offsets[l] integers decoded into out[int_offsets[l]:...] (delta from
        prev[l], default 0).  Offsets are int64 CUDA tensors (n+1 entries);
        ``results`` (optional, int64 CUDA tensor of n*3) receives each list's
        DecodeResult as (status, values_written, bytes_consumed)."""
        n = int(byte_offsets.numel()) - 1
        import torch

        _check_in_tensor(inp, inp.numel())
        for name, t in (("byte_offsets", byte_offsets), ("int_offsets", int_offsets)):
            if not (t.is_cuda and t.dtype == torch.int64 and t.is_contiguous() and t.numel() == n + 1):
                raise MvbError(f"{name} must be a contiguous int64 CUDA tensor of n_lists + 1 entries")
        if prev is not None and not (prev.is_cuda and prev.dtype in (torch.int32, torch.uint32) and
                                     prev.is_contiguous() and prev.numel() >= n):
            raise MvbError("prev must be a contiguous int32/uint32 CUDA tensor of >= n_lists entries")
        if results is not None and not (results.is_cuda and results.dtype == torch.int64 and
                                        results.is_contiguous() and results.numel() >= 3 * n):
            raise MvbError("results must be a contiguous int64 CUDA tensor of >= 3 * n_lists entries")
        if n > 0:
            # the offsets are validated once per tensor object and version (the check
            # reads them back: a device synchronisation that repeated decodes of one
            # batch skip).  Identity, not address: a freed tensor's memory is reused.
            total = None
            for wb, wi, vb, vi, tot in self._lists_ok:
                if wb() is byte_offsets and wi() is int_offsets and vb == byte_offsets._version and \
                        vi == int_offsets._version:
                    total = tot
                    break
            if total is None:
                io_h = int_offsets.cpu()
                if bool((io_h[1:] < io_h[:-1]).any()) or bool((byte_offsets[1:] < byte_offsets[:-1]).any()):
                    raise MvbError("byte_offsets and int_offsets must be non-decreasing")
                total = int(io_h[-1])
                self._lists_ok = [e for e in self._lists_ok if e[0]() is not None and e[1]() is not None][-7:]
                self._lists_ok.append((weakref.ref(byte_offsets), weakref.ref(int_offsets), byte_offsets._version,
                                       int_offsets._version, total))
            _check_out_tensor(out, total, inp.device)
        L = _lib.lib()
        ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        if delta:
            rc = L.mvb_decode_delta_lists_device(ptr(inp) if inp.numel() else None, inp.numel(), byte_offsets.data_ptr(),
                                                 int_offsets.data_ptr(), ptr(prev), n, ptr(order), ptr(out), int(mode),
                                                 ptr(results), self.ws.data_ptr(), self.ws_bytes, self._stream())
        else:
            rc = L.mvb_decode_lists_device(ptr(inp) if inp.numel() else None, inp.numel(), byte_offsets.data_ptr(),
                                           int_offsets.data_ptr(), n, ptr(order), ptr(out), int(mode), ptr(results),
                                           self.ws.data_ptr(), self.ws_bytes, self._stream())
        _check(rc)

    def result(self) -> DecodeResult:
        r = self.res.cpu().numpy().view(np.uint64)
        status = int(np.int64(r[0]) & 0xFFFFFFFF)
        return DecodeResult(DecodeStatus(status), int(r[1]), int(r[2]))


_decoders = {}


def _decoder_for(t) -> Decoder:
    key = t.device.index
    d = _decoders.get(key)
    if d is None:
        d = _decoders[key] = Decoder(t.device)
    return d


def _decode(inp, count, prev, out, options, delta: bool):
    if isinstance(inp, EncodedBuffer):
        inp = inp.bytes
    mode = _mode_of(options)
    count = int(count)
    if _is_cuda_tensor(inp):
        _check_in_tensor(inp, inp.numel())
        _check_out_tensor(out, count, inp.device)
        d = _decoder_for(inp)
        if delta:
            d.decode_delta(inp, count, prev, out, mode)
        else:
            d.decode(inp, count, out, mode)
        return d.result()
    src = _u8(inp)
    if count and (out is None or np.asarray(out).size < count):
        raise MvbError("decode needs an output array with >= count elements")
    dst = out if count else np.zeros(0, np.uint32)
    if not (isinstance(dst, np.ndarray) and dst.dtype in (np.uint32, np.int32) and dst.flags.c_contiguous):
        raise MvbError("output must be a C-contiguous numpy uint32 array")
    res = _lib.MvbResult()
    L = _lib.lib()
    if delta:
        rc = L.mvb_decode_delta_stream(_ptr(src), src.size, count, int(prev) & 0xFFFFFFFF,
                                       _ptr(dst), mode, ctypes.byref(res))
    else:
        rc = L.mvb_decode_stream(_ptr(src), src.size, count, _ptr(dst), mode, ctypes.byref(res))
    _check(rc)
    return DecodeResult(DecodeStatus(res.status), int(res.values_written), int(res.bytes_consumed))


def decode_lists(inp, byte_offsets, int_offsets, out, prev=None, delta: bool = True, results: bool = True):
    """Batched posting lists from host memory (mvb_decode[_delta]_lists): list
    l is inp[byte_offsets[l]:byte_offsets[l+1]] holding int_offsets[l+1] -
    int_offsets[l] integers, decoded (delta from prev[l], default 0) into
    out[int_offsets[l]:...] -- as one decode[_delta]_stream call per list
    (tools/bench/runner.cpp:28-61) would, in one pipelined batch.  Returns the
    per-list DecodeResults as an (n, 3) uint64 array (status, values_written,
    bytes_consumed), or None if ``results`` is False."""
    src = _u8(inp)
    bo = np.ascontiguousarray(byte_offsets, np.uint64)
    io = np.ascontiguousarray(int_offsets, np.uint64)
    n = int(bo.size) - 1
    if io.size != bo.size:
        raise MvbError("byte_offsets and int_offsets need the same length (n_lists + 1)")
    if not (isinstance(out, np.ndarray) and out.dtype in (np.uint32, np.int32) and out.flags.c_contiguous):
        raise MvbError("output must be a C-contiguous numpy uint32 array")
    if n > 0 and (np.any(bo[1:] < bo[:-1]) or np.any(io[1:] < io[:-1])):
        raise MvbError("byte_offsets and int_offsets must be non-decreasing")
    if n > 0 and out.size < int(io[-1]):
        raise MvbError("output array smaller than int_offsets[-1]")
    pv = None if prev is None else np.ascontiguousarray(prev, np.uint32)
    if pv is not None and pv.size < n:
        raise MvbError("prev needs one value per list")
    res = np.zeros((max(n, 1), 3), np.uint64) if results else None
    L = _lib.lib()
    if delta:
        rc = L.mvb_decode_delta_lists(_ptr(src), src.size, _ptr(bo), _ptr(io), _ptr(pv) if pv is not None else None,
                                      n, _ptr(out), 0, _ptr(res) if res is not None else None)
    else:
        rc = L.mvb_decode_lists(_ptr(src), src.size, _ptr(bo), _ptr(io), n, _ptr(out), 0,
                                _ptr(res) if res is not None else None)
    _check(rc)
    if res is None:
        return None
    res[:, 0] &= 0xFFFFFFFF
    return res[:n]


def decode_stream(inp, count=None, out=None, options: Union[DecodeOptions, DecodeMode, int, None] = None):
    """Decodes exactly ``count`` integers of ``inp`` into ``out`` (decode.hpp:44-47).

    ``decode_stream(buf: EncodedBuffer, out, options)`` is the EncodedBuffer
    overload (decode.hpp:46-47)."""
    if isinstance(inp, EncodedBuffer) and (count is None or not np.isscalar(count)):
        inp, count, out, options = inp.bytes, inp.count, count, out
    return _decode(inp, count, 0, out, options, delta=False)


def decode_delta_stream(inp, count=None, prev=0, out=None, options=None):
    """Decodes ``count`` gaps into absolute values starting from ``prev``
    (decode.hpp:51-54).  Overload: ``decode_delta_stream(buf, prev, out, options)``."""
    if isinstance(inp, EncodedBuffer) and not (count is not None and prev is not None and out is not None
                                                and np.isscalar(count) and np.isscalar(prev)):
        inp, count, prev, out, options = inp.bytes, inp.count, count, prev, out
    return _decode(inp, count, prev, out, options, delta=True)


def decode_scalar(inp, count=None, out=None, mode: DecodeMode = DecodeMode.strict):
    """vbyte.hpp:55-58 (same result as decode_stream by definition)."""
    return decode_stream(inp, count, out, mode)


def decode_delta_scalar(inp, count, prev, out, mode: DecodeMode = DecodeMode.strict):
    """vbyte.hpp:62-63."""
    return _decode(inp, count, prev, out, mode, delta=True)


def decode_list(buf, out, buffer_mode: str = "full", buffer_ints: int = 4096, options=None):
    """One delta-coded list, as the reference benchmark runner's decode_list
    (tools/bench/runner.cpp:28-61) does it: "full" decodes the whole list in
    one call; "l1" walks the stream in buffer_ints-integer chunks through a
    reused buffer, carrying bytes_consumed and the running prefix (prev = the
    chunk's last value) into the next call -- the chunked caller pattern the
    drop-in must serve unchanged.  `out` receives the
    whole list (full) or, for l1, each chunk is copied out of the reused
    buffer into it (the reference only keeps the buffer).  Returns the
    DecodeResult of the last call."""
    if not isinstance(buf, EncodedBuffer):
        raise MvbError("decode_list takes an EncodedBuffer")
    if buffer_mode == "full":
        return decode_delta_stream(buf.bytes, buf.count, 0, out, options)
    if buffer_mode != "l1":
        raise MvbError("buffer_mode must be 'full' or 'l1'")
    data = _u8(buf.bytes)
    scratch = np.zeros(max(int(buffer_ints), 1), np.uint32)
    done = offset = 0
    prev = 0
    r = DecodeResult()
    while done < buf.count:
        n = min(int(buffer_ints), buf.count - done)
        r = decode_delta_stream(data[offset:], n, prev, scratch, options)
        if r.status != DecodeStatus.ok:
            return r
        offset += r.bytes_consumed
        prev = int(scratch[n - 1])
        out[done:done + n] = scratch[:n]
        done += n
    return r


def encode_device(values, deltas: bool = False):
    """Device-side encode_sequence / encode_deltas (mvb_encode_*_device) of a
    uint32/int32 CUDA tensor; returns a uint8 CUDA tensor of the encoded
    bytes.  Synchronises to read the length; raises ValueError (as the
    reference's encode_deltas) if `deltas` and the input decreases."""
    import torch

    n = int(values.numel())
    dev = values.device
    L = _lib.lib()
    ws = torch.empty(max(int(L.mvb_encode_workspace_bytes(n)), 8), dtype=torch.uint8, device=dev)
    out = torch.empty(max(5 * n, 1), dtype=torch.uint8, device=dev)
    meta = torch.zeros(2, dtype=torch.int64, device=dev)  # length, first decreasing index
    stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    if deltas:
        _check(L.mvb_encode_deltas_device(values.data_ptr() if n else None, n, out.data_ptr(), meta.data_ptr(),
                                          meta.data_ptr() + 8, ws.data_ptr(), ws.numel(), stream))
    else:
        _check(L.mvb_encode_sequence_device(values.data_ptr() if n else None, n, out.data_ptr(), meta.data_ptr(),
                                            ws.data_ptr(), ws.numel(), stream))
    m = meta.cpu().numpy().view(np.uint64)
    if deltas and n and int(m[1]) != 0xFFFFFFFFFFFFFFFF:
        raise ValueError(f"encode_deltas: input decreases at index {int(m[1])}")
    return out[:int(m[0])]


def version() -> str:
    return _lib.lib().mvb_version().decode()
