"""ctypes binding of the C ABI in include/mvb_cuda.h (libmvb_cuda.so).

The shared library is built in-tree by ``paper_1503_07387_b200.build`` (nvcc,
sm_100a).  There is no fallback: importing the decoder without the library
raises, so a missing build can never silently turn into a CPU path.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MVB_CUDA_LIB") or os.path.join(HERE, "libmvb_cuda.so")  # override: experiments only
WORKLOAD_LIB_PATH = os.path.join(HERE, "libmvb_workload.so")

# Every symbol include/mvb_cuda.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "mvb_workspace_bytes",
    "mvb_workspace_init",
    "mvb_decode_device",
    "mvb_decode_delta_device",
    "mvb_delta_totals_device",
    "mvb_decode_delta_totaled_device",
    "mvb_shard_cuts",
    "mvb_decode_delta_sharded",
    "mvb_decode_delta_device_dprev",
    "mvb_shard_carry_device",
    "mvb_decode_lists_device",
    "mvb_decode_delta_lists_device",
    "mvb_decode_lists",
    "mvb_decode_delta_lists",
    "mvb_encode_workspace_bytes",
    "mvb_encode_sequence_device",
    "mvb_encode_deltas_device",
    "mvb_decode_stream",
    "mvb_decode_delta_stream",
    "mvb_encoded_size",
    "mvb_encode_one",
    "mvb_encoded_length",
    "mvb_encode_sequence",
    "mvb_encode_deltas",
    "mvb_version",
)


class MvbResult(ctypes.Structure):
    """mvb_result: layout of mvb::DecodeResult (vbyte.hpp:45-49) across the ABI."""

    _fields_ = [
        ("status", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("values_written", ctypes.c_uint64),
        ("bytes_consumed", ctypes.c_uint64),
    ]


_lib = None
_wlib = None

c_u8p = ctypes.c_void_p
c_size = ctypes.c_size_t


def _declare(lib):
    vp, sz, u32, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_int
    lib.mvb_workspace_bytes.argtypes = [sz]
    lib.mvb_workspace_bytes.restype = sz
    lib.mvb_workspace_init.argtypes = [vp, sz, vp]
    lib.mvb_workspace_init.restype = i32
    lib.mvb_decode_device.argtypes = [vp, sz, sz, vp, i32, vp, vp, sz, vp]
    lib.mvb_decode_device.restype = i32
    lib.mvb_decode_delta_device.argtypes = [vp, sz, sz, u32, vp, i32, vp, vp, sz, vp]
    lib.mvb_decode_delta_device.restype = i32
    lib.mvb_decode_delta_device_dprev.argtypes = [vp, sz, sz, vp, vp, i32, vp, vp, sz, vp]
    lib.mvb_decode_delta_device_dprev.restype = i32
    lib.mvb_shard_carry_device.argtypes = [vp, i32, i32, i32, u32, vp, vp, vp]
    lib.mvb_shard_carry_device.restype = i32
    lib.mvb_decode_lists_device.argtypes = [vp, sz, vp, vp, sz, vp, vp, i32, vp, vp, sz, vp]
    lib.mvb_decode_lists_device.restype = i32
    lib.mvb_decode_delta_lists_device.argtypes = [vp, sz, vp, vp, vp, sz, vp, vp, i32, vp, vp, sz, vp]
    lib.mvb_decode_delta_lists_device.restype = i32
    lib.mvb_decode_lists.argtypes = [vp, sz, vp, vp, sz, vp, i32, vp]
    lib.mvb_decode_lists.restype = i32
    lib.mvb_decode_delta_lists.argtypes = [vp, sz, vp, vp, vp, sz, vp, i32, vp]
    lib.mvb_decode_delta_lists.restype = i32
    lib.mvb_encode_workspace_bytes.argtypes = [sz]
    lib.mvb_encode_workspace_bytes.restype = sz
    lib.mvb_encode_sequence_device.argtypes = [vp, sz, vp, vp, vp, sz, vp]
    lib.mvb_encode_sequence_device.restype = i32
    lib.mvb_encode_deltas_device.argtypes = [vp, sz, vp, vp, vp, vp, sz, vp]
    lib.mvb_encode_deltas_device.restype = i32
    lib.mvb_decode_stream.argtypes = [vp, sz, sz, vp, i32, ctypes.POINTER(MvbResult)]
    lib.mvb_decode_stream.restype = i32
    lib.mvb_decode_delta_stream.argtypes = [vp, sz, sz, u32, vp, i32, ctypes.POINTER(MvbResult)]
    lib.mvb_decode_delta_stream.restype = i32
    lib.mvb_encoded_size.argtypes = [u32]
    lib.mvb_encoded_size.restype = sz
    lib.mvb_encode_one.argtypes = [u32, vp]
    lib.mvb_encode_one.restype = sz
    lib.mvb_encoded_length.argtypes = [vp, sz]
    lib.mvb_encoded_length.restype = sz
    lib.mvb_encode_sequence.argtypes = [vp, sz, vp]
    lib.mvb_encode_sequence.restype = sz
    lib.mvb_encode_deltas.argtypes = [vp, sz, vp, ctypes.POINTER(sz), ctypes.POINTER(sz)]
    lib.mvb_encode_deltas.restype = i32
    if hasattr(lib, "mvb_delta_totals_device"):  # (older builds under MVB_CUDA_LIB lack the sharded entries)
        lib.mvb_delta_totals_device.argtypes = [vp, sz, vp, vp, sz, vp]
        lib.mvb_delta_totals_device.restype = i32
        lib.mvb_decode_delta_totaled_device.argtypes = [vp, sz, sz, u32, vp, vp, vp, vp, sz, vp]
        lib.mvb_decode_delta_totaled_device.restype = i32
        lib.mvb_shard_cuts.argtypes = [vp, sz, i32, vp]
        lib.mvb_shard_cuts.restype = i32
        lib.mvb_decode_delta_sharded.argtypes = [i32, vp, vp, vp, sz, u32, vp, vp, ctypes.POINTER(MvbResult)]
        lib.mvb_decode_delta_sharded.restype = i32
    lib.mvb_version.argtypes = []
    lib.mvb_version.restype = ctypes.c_char_p
    return lib


def lib():
    """The loaded libmvb_cuda.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the CUDA decoder has no CPU fallback)")
        _lib = _declare(ctypes.CDLL(LIB_PATH))
    return _lib


def kernels_per_decode(mode: int = 0) -> int:
    """Kernels one decode call launches in steady state (internal symbol)."""
    f = lib().mvbx_kernels_per_decode
    f.argtypes = [ctypes.c_int]
    f.restype = ctypes.c_int
    return int(f(int(mode)))


def set_kernel_choice(choice: int) -> None:
    """Testing switch (internal symbol mvbx_set_kernel): strict-mode stream
    decoder 0 = the single-read fused decoder (default), 1 = the per-tile
    kernel (which serves permissive mode), 6 = the two-kernel segmented
    decoder (whose launch pair the pipelined host drop-in uses).  Batched
    lists have one kernel."""
    f = lib().mvbx_set_kernel
    f.argtypes = [ctypes.c_int]
    f.restype = None
    f(int(choice))


def set_host_pipeline(min_bytes: int = 4 << 20, chunk_bytes: int = 1 << 20, grow: bool = True) -> None:
    """Testing switch (internal symbol mvbx_set_host_pipeline): the host
    drop-ins (mvb_decode_stream / mvb_decode_delta_stream, strict mode) decode
    streams of at least `min_bytes` scanned bytes in chunks (whole 32-segment
    groups), the first of about `chunk_bytes`, later ones doubling up to 16 MB
    if `grow`, overlapping H2D, decode and D2H; the defaults are the
    library's."""
    f = lib().mvbx_set_host_pipeline
    f.argtypes = [ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int]
    f.restype = None
    f(int(min_bytes), int(chunk_bytes), int(bool(grow)))


def workload_lib():
    """Host-side generators/encoder used to build bench and test inputs."""
    global _wlib
    if _wlib is None:
        if not os.path.exists(WORKLOAD_LIB_PATH):
            raise RuntimeError(f"{WORKLOAD_LIB_PATH} is missing: run the build first")
        w = ctypes.CDLL(WORKLOAD_LIB_PATH)
        vp, sz, u32, u64, dbl = (ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32,
                                 ctypes.c_uint64, ctypes.c_double)
        w.mvbw_mixed_values.argtypes = [vp, sz, u32]
        w.mvbw_mixture.argtypes = [vp, sz, u64, dbl, u32, u32, u32, u32]
        w.mvbw_geometric_gaps.argtypes = [vp, sz, u64, dbl, dbl, u32, u32]
        w.mvbw_loguniform_lengths.argtypes = [vp, sz, u64, u32, u32]
        w.mvbw_clustered_lists.argtypes = [vp, vp, vp, sz, u64, u64]
        w.mvbw_encoded_length.argtypes = [vp, sz]
        w.mvbw_encoded_length.restype = sz
        w.mvbw_encode.argtypes = [vp, sz, vp]
        w.mvbw_encode.restype = sz
        w.mvbw_delta.argtypes = [vp, sz, vp]
        w.mvbw_delta.restype = sz
        w.mvbw_delta_lists.argtypes = [vp, vp, sz, vp]
        for f in ("mvbw_mixed_values", "mvbw_mixture", "mvbw_geometric_gaps",
                  "mvbw_loguniform_lengths", "mvbw_clustered_lists", "mvbw_delta_lists"):
            getattr(w, f).restype = None
        _wlib = w
    return _wlib
