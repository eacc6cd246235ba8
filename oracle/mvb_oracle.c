/*
 * oracle/mvb_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's conventional (scalar) VByte codec,
 * used as the parity checker for the CUDA decoder.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this
 * library; the product path (paper_1503_07387_b200/) never links or calls it.
 *
 * Parity pin: tests/test_oracle.py checks every function here against the
 * reference library itself (oracle/_ref/libmvb_ref.so, built from
 * /root/reference/proj/core/src by oracle/Makefile) and against the golden
 * vectors committed under tests/golden/.
 *
 * Reference anchors (paths relative to /root/reference/proj):
 *   wire format      core/include/mvb/vbyte.hpp:10-20
 *   encoded_size     core/src/vbyte.cpp:9-15
 *   encode_one       core/src/vbyte.cpp:17-25
 *   encode_sequence  core/src/vbyte.cpp:33-39
 *   one integer      core/src/internal.hpp:22-37 (strict 5th-byte rule :35,
 *                    mod-2^32 wrap :36)
 *   decode_scalar    core/src/vbyte.cpp:47-57
 *   decode_delta     core/src/vbyte.cpp:63-74
 *   delta_encode     core/src/vbyte.cpp:76-86
 *   prefix_sum       core/src/vbyte.cpp:88-93
 */
#include <stddef.h>
#include <stdint.h>

enum { OR_OK = 0, OR_TRUNCATED = 1, OR_MALFORMED = 2 };
enum { OR_STRICT = 0, OR_PERMISSIVE = 1 };

typedef struct {
    int32_t status;
    int32_t pad;
    uint64_t values_written;
    uint64_t bytes_consumed;
} oracle_result;

/* vbyte.cpp:9-15 */
size_t oracle_encoded_size(uint32_t x) {
    size_t n = 1;
    while (n < 5 && (x >> (7 * n)) != 0) ++n;
    return n;
}

/* vbyte.cpp:17-25: low 7-bit digit first, 0x80 on all but the last byte. */
size_t oracle_encode_one(uint32_t x, uint8_t *out) {
    size_t n = oracle_encoded_size(x);
    for (size_t k = 0; k < n; ++k) {
        uint8_t digit = (uint8_t)((x >> (7 * k)) & 0x7F);
        out[k] = (uint8_t)(k + 1 < n ? (digit | 0x80) : digit);
    }
    return n;
}

/* vbyte.cpp:33-39; returns bytes written (caller sizes out >= 5n). */
size_t oracle_encode_sequence(const uint32_t *v, size_t n, uint8_t *out) {
    size_t pos = 0;
    for (size_t i = 0; i < n; ++i) pos += oracle_encode_one(v[i], out + pos);
    return pos;
}

/* Exact byte count of encode_sequence(v). */
size_t oracle_encoded_length(const uint32_t *v, size_t n) {
    size_t total = 0;
    for (size_t i = 0; i < n; ++i) total += oracle_encoded_size(v[i]);
    return total;
}

/*
 * internal.hpp:22-37.  Returns consumed bytes (1..5) or 0 on error with
 * *status set.  The fifth byte is taken whole and the value wraps mod 2^32;
 * strict mode rejects a fifth byte >= 0x10.
 */
static unsigned one_int(const uint8_t *p, size_t avail, int mode, uint32_t *value, int *status) {
    uint32_t acc = 0;
    for (unsigned k = 0; k < 4; ++k) {
        if (k >= avail) { *status = OR_TRUNCATED; return 0; }
        uint32_t b = p[k];
        if (b < 0x80) { *value = acc | (b << (7 * k)); *status = OR_OK; return k + 1; }
        acc |= (b & 0x7F) << (7 * k);
    }
    if (avail < 5) { *status = OR_TRUNCATED; return 0; }
    uint32_t b = p[4];
    if (mode == OR_STRICT && b >= 0x10) { *status = OR_MALFORMED; return 0; }
    *value = acc + (b << 28); /* unsigned arithmetic: mod 2^32 */
    *status = OR_OK;
    return 5;
}

/* vbyte.cpp:47-57 (delta=0) and :63-74 (delta=1: prev += v; out[i] = prev). */
static oracle_result decode_impl(const uint8_t *in, size_t len, size_t count, uint32_t *out,
                                 int mode, int delta, uint32_t prev) {
    oracle_result r = {OR_OK, 0, 0, 0};
    size_t pos = 0;
    for (size_t i = 0; i < count; ++i) {
        uint32_t v = 0;
        int st = OR_OK;
        unsigned used = one_int(in + pos, len - pos, mode, &v, &st);
        if (st != OR_OK) {
            r.status = st;
            r.values_written = i;
            r.bytes_consumed = pos;
            return r;
        }
        if (delta) { prev += v; v = prev; }
        out[i] = v;
        pos += used;
    }
    r.values_written = count;
    r.bytes_consumed = pos;
    return r;
}

oracle_result oracle_decode(const uint8_t *in, size_t len, size_t count, uint32_t *out, int mode) {
    return decode_impl(in, len, count, out, mode, 0, 0);
}

oracle_result oracle_decode_delta(const uint8_t *in, size_t len, size_t count, uint32_t prev,
                                  uint32_t *out, int mode) {
    return decode_impl(in, len, count, out, mode, 1, prev);
}

/* vbyte.cpp:76-86.  Returns -1 (and leaves gaps partially written) when the
 * input decreases at some index; that index is stored in *bad_index. */
int oracle_delta_encode(const uint32_t *values, size_t n, uint32_t *gaps, size_t *bad_index) {
    uint32_t prev = 0;
    for (size_t i = 0; i < n; ++i) {
        if (values[i] < prev) { if (bad_index) *bad_index = i; return -1; }
        gaps[i] = values[i] - prev;
        prev = values[i];
    }
    return 0;
}

/* vbyte.cpp:88-93; in-place allowed. */
void oracle_prefix_sum(const uint32_t *gaps, size_t n, uint32_t prev, uint32_t *out) {
    for (size_t i = 0; i < n; ++i) { prev += gaps[i]; out[i] = prev; }
}

/* FNV-1a over the little-endian bytes of a u32 array (tools/bench/runner.cpp:63-72). */
uint64_t oracle_fnv1a_u32(const uint32_t *data, size_t n, uint64_t hash) {
    for (size_t i = 0; i < n; ++i) {
        uint32_t v = data[i];
        for (int b = 0; b < 4; ++b, v >>= 8) { hash ^= v & 0xFF; hash *= 0x100000001B3ull; }
    }
    return hash;
}

uint64_t oracle_fnv1a_bytes(const uint8_t *data, size_t n, uint64_t hash) {
    for (size_t i = 0; i < n; ++i) { hash ^= data[i]; hash *= 0x100000001B3ull; }
    return hash;
}
