// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference library (mvbyte), compiled by
// oracle/Makefile together with the reference sources where they lie under
// /root/reference/proj/core/src, into oracle/_ref/libmvb_ref.so.  It is the
// pin for oracle/mvb_oracle.c and the "reference" CPU arm of bench.py.  No
// reference source is copied into this repository.
//
// Each entry forwards to the reference symbol named beside it
// (paths relative to /root/reference/proj):
//   mvbref_encode_sequence     core/src/vbyte.cpp:33-39
//   mvbref_encode_deltas       core/src/vbyte.cpp:41-45
//   mvbref_decode_scalar       core/src/vbyte.cpp:47-57
//   mvbref_decode_delta_scalar core/src/vbyte.cpp:63-74
//   mvbref_decode_stream       core/src/decode.cpp:73-82  (auto path: SSE if present)
//   mvbref_decode_delta_stream core/src/decode.cpp:88-97
//   mvbref_vector_available    core/src/decode.cpp:28-34
//   mvbref_write_list_file     core/src/list_file.cpp:57-65
//   mvbref_read_list_file      core/src/list_file.cpp:89-93 (-1 on ListFileError)
//   mvbref_decode_delta_lists  one decode_delta_stream call per list, as
//                              tools/bench/runner.cpp:28-61 decode_list does
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <vector>

#include "mvb/decode.hpp"
#include "mvb/list_file.hpp"
#include "mvb/vbyte.hpp"

extern "C" {

struct mvbref_result {
    int32_t status;
    int32_t pad;
    uint64_t values_written;
    uint64_t bytes_consumed;
};

static mvbref_result pack(const mvb::DecodeResult& r) {
    return {static_cast<int32_t>(r.status), 0, r.values_written, r.bytes_consumed};
}

static mvb::DecodeOptions opts(int mode, int path, size_t handoff) {
    mvb::DecodeOptions o;
    o.mode = mode ? mvb::DecodeMode::permissive : mvb::DecodeMode::strict;
    o.path = path == 1 ? mvb::DecodePath::portable
             : path == 2 ? mvb::DecodePath::vector
                         : mvb::DecodePath::auto_select;
    if (handoff) o.scalar_handoff = handoff;
    return o;
}

int mvbref_vector_available() { return mvb::vector_path_available() ? 1 : 0; }

// Returns encoded length; writes into out when out != nullptr (caller sizes it
// with a first call passing out = nullptr).
size_t mvbref_encode_sequence(const uint32_t* v, size_t n, uint8_t* out) {
    mvb::EncodedBuffer b = mvb::encode_sequence(std::span<const uint32_t>(v, n));
    if (out) std::memcpy(out, b.bytes.data(), b.bytes.size());
    return b.bytes.size();
}

// Returns encoded length, or (size_t)-1 when the reference throws
// std::invalid_argument (decreasing input).
size_t mvbref_encode_deltas(const uint32_t* v, size_t n, uint8_t* out) {
    try {
        mvb::EncodedBuffer b = mvb::encode_deltas(std::span<const uint32_t>(v, n));
        if (out) std::memcpy(out, b.bytes.data(), b.bytes.size());
        return b.bytes.size();
    } catch (const std::invalid_argument&) {
        return static_cast<size_t>(-1);
    }
}

mvbref_result mvbref_decode_scalar(const uint8_t* in, size_t len, size_t count, uint32_t* out,
                                   int mode) {
    return pack(mvb::decode_scalar(std::span<const uint8_t>(in, len), count, out,
                                   mode ? mvb::DecodeMode::permissive : mvb::DecodeMode::strict));
}

mvbref_result mvbref_decode_delta_scalar(const uint8_t* in, size_t len, size_t count,
                                         uint32_t prev, uint32_t* out, int mode) {
    return pack(mvb::decode_delta_scalar(
        std::span<const uint8_t>(in, len), count, prev, out,
        mode ? mvb::DecodeMode::permissive : mvb::DecodeMode::strict));
}

mvbref_result mvbref_decode_stream(const uint8_t* in, size_t len, size_t count, uint32_t* out,
                                   int mode, int path, size_t handoff) {
    return pack(mvb::decode_stream(std::span<const uint8_t>(in, len), count, out,
                                   opts(mode, path, handoff)));
}

mvbref_result mvbref_decode_delta_stream(const uint8_t* in, size_t len, size_t count,
                                         uint32_t prev, uint32_t* out, int mode, int path,
                                         size_t handoff) {
    return pack(mvb::decode_delta_stream(std::span<const uint8_t>(in, len), count, prev, out,
                                         opts(mode, path, handoff)));
}

int mvbref_write_list_file(const char* path, const uint8_t* bytes, size_t len, uint32_t count, int delta) {
    try {
        mvb::EncodedBuffer b;
        b.bytes.assign(bytes, bytes + len);
        b.count = count;
        b.delta_coded = delta != 0;
        mvb::write_list_file(path, b);
        return 0;
    } catch (const mvb::ListFileError&) {
        return 1;
    }
}

// Payload length (bytes copied into out, up to cap), or -1 on ListFileError.
long long mvbref_read_list_file(const char* path, int validate, uint8_t* out, size_t cap, uint32_t* count,
                                int* delta) {
    try {
        const mvb::EncodedBuffer b = mvb::read_list_file(path, validate != 0);
        *count = b.count;
        *delta = b.delta_coded ? 1 : 0;
        std::memcpy(out, b.bytes.data(), std::min(cap, b.bytes.size()));
        return static_cast<long long>(b.bytes.size());
    } catch (const mvb::ListFileError&) {
        return -1;
    }
}

// Lists [lo, hi) of a batch (byte / integer offsets, n_lists + 1 entries):
// the reference's per-list loop; returns the number of lists not OK.
size_t mvbref_decode_delta_lists(const uint8_t* in, const uint64_t* byte_off, const uint64_t* int_off,
                                 uint32_t* out, size_t lo, size_t hi) {
    size_t bad = 0;
    for (size_t l = lo; l < hi; ++l) {
        const auto r = mvb::decode_delta_stream(
            std::span<const uint8_t>(in + byte_off[l], byte_off[l + 1] - byte_off[l]),
            int_off[l + 1] - int_off[l], 0, out + int_off[l], mvb::DecodeOptions{});
        if (r.status != mvb::DecodeStatus::ok) ++bad;
    }
    return bad;
}

}  // extern "C"
