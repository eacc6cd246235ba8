"""B200-native VByte codec (arxiv 1503.07387 "Masked VByte" decode path).

The decoder is hand-written sm_100a CUDA behind the C ABI in
include/mvb_cuda.h; this package is the Python mirror of the reference's
codec interface (see ``mvb``) plus the multi-GPU sharded decode (``shard``)
and the synthetic workloads of BASELINE.json (``workload``).
"""
from .mvb import (  # noqa: F401
    Decoder,
    DecodeMode,
    DecodeOptions,
    DecodePath,
    DecodeResult,
    DecodeStatus,
    EncodedBuffer,
    MvbError,
    decode_delta_scalar,
    decode_delta_stream,
    decode_scalar,
    decode_stream,
    delta_encode,
    encode_deltas,
    encode_one,
    encode_sequence,
    encoded_size,
    prefix_sum_scalar,
    version,
)
