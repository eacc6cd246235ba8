/*
 * mvb_cuda.h -- C ABI of the B200-native VByte codec (libmvb_cuda.so).
 *
 * Drop-in boundary for the reference's decode path (arxiv 1503.07387,
 * "Masked VByte"; reference library `mvbyte`, paths relative to
 * /root/reference/proj).  Each entry point names the reference interface it
 * replaces.  Semantics (outputs, DecodeStatus, values_written,
 * bytes_consumed, strict/permissive) are those of the reference's documented
 * oracle decode_scalar / decode_delta_scalar (core/include/mvb/vbyte.hpp:51-63),
 * which decode_stream / decode_delta_stream promise to equal on every
 * canonical stream (core/include/mvb/decode.hpp:42-54).
 *
 * Conventions
 *   - Data errors are status values, never crashes: MVB_OK / MVB_TRUNCATED /
 *     MVB_MALFORMED mirror mvb::DecodeStatus (vbyte.hpp:43).  API misuse and
 *     CUDA failures are negative return codes (the reference throws there:
 *     decode.cpp:55-56, vbyte.cpp:80-81); no exception crosses this ABI.
 *   - The caller owns every buffer.  Decoders never read past in + in_len and
 *     never write past out + count.  On a non-OK status,
 *     out[values_written .. count) is unspecified (the reference's vector path
 *     may also store past the last value it reports, stream_loop.hpp:28-29).
 *   - count == 0 is valid with out == NULL (decode_test.cpp:204-206).
 *   - "_device" entry points take device pointers and run asynchronously on
 *     `stream`; they allocate nothing.  Their result lands in device memory
 *     (res_dev, may be NULL) so back-to-back calls need no host sync.
 *   - Host-pointer entry points (mvb_decode_stream, ...) are synchronous
 *     drop-ins for the reference functions of the same name: they copy
 *     in -> device, decode, copy out -> host on an internal stream, using
 *     device buffers cached per calling thread.
 *   - Reentrant per (stream, workspace).  No global mutable state except the
 *     host wrappers' per-thread buffer cache.
 */
#ifndef MVB_CUDA_H
#define MVB_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *mvb_stream_t; /* == cudaStream_t */

/* mvb::DecodeStatus (vbyte.hpp:43) */
enum {
    MVB_OK = 0,
    MVB_TRUNCATED = 1,
    MVB_MALFORMED = 2
};

/* API errors (negative) */
enum {
    MVB_ERR_INVALID_ARG = -1, /* null pointer with nonzero size, bad mode, ... */
    MVB_ERR_WORKSPACE = -2,   /* workspace missing or smaller than mvb_workspace_bytes() */
    MVB_ERR_CUDA = -3,        /* a CUDA runtime call failed */
    MVB_ERR_DECREASING = -4   /* mvb_encode_deltas: input decreases (vbyte.cpp:80-81) */
};

/* mvb::DecodeMode (vbyte.hpp:38-41) */
enum {
    MVB_STRICT = 0,    /* reject a fifth byte >= 0x10 */
    MVB_PERMISSIVE = 1 /* take the fifth byte whole, value mod 2^32 */
};

/* mvb::DecodeResult (vbyte.hpp:45-49); 24 bytes, same layout on host and device. */
typedef struct {
    int32_t status;
    int32_t reserved;
    uint64_t values_written;
    uint64_t bytes_consumed;
} mvb_result;

/* ---------------------------------------------------------------- device API */

/* Bytes of device workspace a decode of in_len input bytes needs.  The
 * workspace must be zeroed once (mvb_workspace_init or cudaMemset 0) before
 * its first use; afterwards each decode leaves it ready for the next. */
size_t mvb_workspace_bytes(size_t in_len);
int mvb_workspace_init(void *ws, size_t ws_bytes, mvb_stream_t stream);

/* Replaces mvb::decode_stream (decode.hpp:44-45, decode.cpp:73-82) and
 * mvb::decode_scalar (vbyte.hpp:55-56, vbyte.cpp:47-57).
 * Decodes exactly `count` integers from in[0..in_len) into out[0..count).
 * Returns 0 when the launch was queued (the decode status is in *res_dev),
 * or a negative MVB_ERR_*. */
int mvb_decode_device(const uint8_t *in, size_t in_len, size_t count, uint32_t *out, int mode,
                      mvb_result *res_dev, void *ws, size_t ws_bytes, mvb_stream_t stream);

/* Replaces mvb::decode_delta_stream (decode.hpp:51-52, decode.cpp:88-97) and
 * mvb::decode_delta_scalar (vbyte.hpp:62-63, vbyte.cpp:63-74): decodes
 * `count` gaps and writes out[i] = prev + gap[0] + ... + gap[i] (mod 2^32). */
int mvb_decode_delta_device(const uint8_t *in, size_t in_len, size_t count, uint32_t prev,
                            uint32_t *out, int mode, mvb_result *res_dev, void *ws,
                            size_t ws_bytes, mvb_stream_t stream);

/* mvb_decode_delta_device with the starting value read from device memory
 * when the kernel runs (prev = *prev_dev), so a carry computed on the device
 * (mvb_shard_carry_device) feeds the decode without a host round trip. */
int mvb_decode_delta_device_dprev(const uint8_t *in, size_t in_len, size_t count,
                                  const uint32_t *prev_dev, uint32_t *out, int mode,
                                  mvb_result *res_dev, void *ws, size_t ws_bytes,
                                  mvb_stream_t stream);

/* Seam fix-up of the sharded decode: from n_ranks all-gathered records of
 * record_words u64 each (word 0 = integer count, low 32 bits of word 1 = gap
 * sum, as written by mvb_delta_totals_device), writes shard `rank`'s carry-in
 * prev + sum[0..rank) mod 2^32 and its output offset count[0..rank).  Either
 * output may be NULL.  Asynchronous on `stream`. */
int mvb_shard_carry_device(const unsigned long long *records, int n_ranks, int rank,
                           int record_words, uint32_t prev, uint32_t *carry_dev,
                           unsigned long long *offset_dev, mvb_stream_t stream);

/* Batched posting lists (BASELINE config 3).  The reference
 * decodes a batch with one decode_delta_stream call per list
 * (tools/bench/runner.cpp:28-61); this decodes them all in one launch, one
 * warp per list.  List l is the byte span in[byte_off[l] .. byte_off[l+1])
 * holding int_off[l+1] - int_off[l] integers; they land in
 * out[int_off[l] .. int_off[l+1]), decoded as decode_stream /
 * decode_delta_stream(span, count, prev[l] (0 if prev == NULL), ...) would,
 * and results[l] (may be NULL) receives that call's DecodeResult.  byte_off,
 * int_off (n_lists + 1 entries each), prev, order and results are device
 * arrays; order (may be NULL) is the order lists are handed out in (longest
 * first balances best).  Strict mode only (MVB_ERR_INVALID_ARG otherwise:
 * decode permissive lists one by one).  The workspace needs only the header
 * (mvb_workspace_bytes(0)).  Asynchronous on `stream`. */
int mvb_decode_lists_device(const uint8_t *in, size_t in_len, const unsigned long long *byte_off,
                            const unsigned long long *int_off, size_t n_lists, const unsigned *order,
                            uint32_t *out, int mode, mvb_result *results, void *ws, size_t ws_bytes,
                            mvb_stream_t stream);
int mvb_decode_delta_lists_device(const uint8_t *in, size_t in_len, const unsigned long long *byte_off,
                                  const unsigned long long *int_off, const uint32_t *prev,
                                  size_t n_lists, const unsigned *order, uint32_t *out, int mode,
                                  mvb_result *results, void *ws, size_t ws_bytes, mvb_stream_t stream);

/* Host-pointer batched decode (the same lists, offsets and results as the
 * _device entry points above, all in host memory).  Synchronous.  The lists
 * are cut into contiguous sub-batches whose host->device copies, decodes and
 * device->host copies overlap (each sub-batch's output range is known from
 * int_off, so no host round trip sits between them); pinned buffers make the
 * copies asynchronous.  Strict mode only.  Returns 0 or a negative MVB_ERR_*;
 * the per-list statuses are in results[] (may be NULL). */
int mvb_decode_lists(const uint8_t *in, size_t in_len, const unsigned long long *byte_off,
                     const unsigned long long *int_off, size_t n_lists, uint32_t *out, int mode,
                     mvb_result *results);
int mvb_decode_delta_lists(const uint8_t *in, size_t in_len, const unsigned long long *byte_off,
                           const unsigned long long *int_off, const uint32_t *prev, size_t n_lists,
                           uint32_t *out, int mode, mvb_result *results);

/* ------------------------------------------------------ sharded delta decode */

/* A delta stream split by byte range over several GPUs (SURVEY.md §8e,
 * BASELINE.json config 4): each shard's decode needs the gap sum of the
 * shards before it.  The reference decodes one stream on one thread
 * (decode.hpp:51-52); these split its decode_delta_stream.
 *
 * mvb_delta_totals_device: one read of in (the single-read decoder's totals
 * pass, last unit first): rec_dev[0] = integers in in, rec_dev[1] = the sum
 * of their values mod 2^32 (the gap sum).  The workspace keeps the per-unit
 * totals for the decode pass: mvb_decode_delta_totaled_device must follow on
 * the same stream with the same in, in_len and workspace (strict mode; it
 * reads in again, the units the totals pass read last from L2).
 * mvb_decode_delta_totaled_device: decode_delta_stream(in, count, prev +
 * (prev_dev ? *prev_dev : 0)) with the totals already known. */
int mvb_delta_totals_device(const uint8_t *in, size_t in_len, unsigned long long *rec_dev, void *ws,
                            size_t ws_bytes, mvb_stream_t stream);
int mvb_decode_delta_totaled_device(const uint8_t *in, size_t in_len, size_t count, uint32_t prev,
                                    const uint32_t *prev_dev, uint32_t *out, mvb_result *res_dev, void *ws,
                                    size_t ws_bytes, mvb_stream_t stream);

/* Cut in (host bytes) into n shards at integer boundaries: cuts[0] = 0,
 * cuts[n] = in_len, cuts[g] = the first integer start at or after
 * in_len * g / n (a continuation run with no end stays whole in shard g-1). */
int mvb_shard_cuts(const uint8_t *in, size_t in_len, int n, unsigned long long *cuts);

/* decode_delta_stream(in, count, prev, out) of one stream held as n shards
 * on n GPUs of this process (devices[g] may repeat: several shards on one
 * GPU).  shard_in[g] / shard_len[g]: shard g's bytes, a device pointer on
 * devices[g] -- consecutive pieces of the stream cut at integer boundaries
 * (mvb_shard_cuts).  Shard g's values go to shard_out[g] (device, room for
 * shard_len[g] values) and are out[offsets[g] ...] of the whole decode.  The
 * shards but the last are totalled (one read each, concurrently), the 16-byte
 * totals exchanged, then every shard decodes from its carry.  Returns the
 * whole stream's DecodeResult (status; *res may be NULL), synchronously. */
int mvb_decode_delta_sharded(int n, const int *devices, const uint8_t *const *shard_in, const size_t *shard_len,
                             size_t count, uint32_t prev, uint32_t *const *shard_out, unsigned long long *offsets,
                             mvb_result *res);

/* ------------------------------------------------------------ host drop-ins */

/* Synchronous host-pointer equivalents of decode_stream / decode_delta_stream
 * (and of decode_scalar / decode_delta_scalar, which have identical results).
 * Return value: the DecodeStatus (>= 0) or a negative MVB_ERR_*; *res (may be
 * NULL) receives the full DecodeResult.  Strict-mode streams of >= 4 MB are
 * decoded in chunks that overlap the host->device copy of later chunks, the
 * decode and the device->host copy of earlier chunks' values (pinned buffers
 * make the copies asynchronous; pageable ones still work).  Only
 * out[0 .. values_written) (and, after a malformed integer, possibly a few
 * more decoded slots) is written. */
int mvb_decode_stream(const uint8_t *in, size_t in_len, size_t count, uint32_t *out, int mode,
                      mvb_result *res);
int mvb_decode_delta_stream(const uint8_t *in, size_t in_len, size_t count, uint32_t prev,
                            uint32_t *out, int mode, mvb_result *res);

/* ------------------------------------------------------------------ encoder */

/* vbyte.cpp:9-15 */
size_t mvb_encoded_size(uint32_t x);
/* vbyte.cpp:17-25: writes 1..5 bytes, returns the count. */
size_t mvb_encode_one(uint32_t x, uint8_t *out);
/* vbyte.cpp:33-39 (host): returns bytes written; out needs
 * mvb_encoded_length(values, n) bytes (<= 5n). */
size_t mvb_encoded_length(const uint32_t *values, size_t n);
size_t mvb_encode_sequence(const uint32_t *values, size_t n, uint8_t *out);
/* vbyte.cpp:41-45 (host): delta_encode + encode_sequence.  Returns 0 and sets
 * *out_len, or MVB_ERR_DECREASING (and *bad_index) if values decreases. */
int mvb_encode_deltas(const uint32_t *sorted_values, size_t n, uint8_t *out, size_t *out_len,
                      size_t *bad_index);

/* Device-side encoder (vbyte.cpp:17-45).  Encodes n
 * device values into out (device, capacity >= 5n bytes, or the exact length
 * from a previous call) and writes the byte count to *len_dev.  The workspace
 * (any contents) must hold mvb_encode_workspace_bytes(n) bytes.  Asynchronous
 * on `stream`.  The deltas form encodes the gaps x[i] - x[i-1] (x[-1] = 0) and
 * writes to *bad_index_dev the first index where the input decreases, or
 * ~0ull if it never does (the reference throws std::invalid_argument there,
 * vbyte.cpp:80-81; the encoded bytes are then unspecified). */
size_t mvb_encode_workspace_bytes(size_t n);
int mvb_encode_sequence_device(const uint32_t *values, size_t n, uint8_t *out, unsigned long long *len_dev,
                               void *ws, size_t ws_bytes, mvb_stream_t stream);
int mvb_encode_deltas_device(const uint32_t *sorted_values, size_t n, uint8_t *out,
                             unsigned long long *len_dev, unsigned long long *bad_index_dev, void *ws,
                             size_t ws_bytes, mvb_stream_t stream);

/* Library build/version string. */
const char *mvb_version(void);

#ifdef __cplusplus
}
#endif

#endif /* MVB_CUDA_H */
