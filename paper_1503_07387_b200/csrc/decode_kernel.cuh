// decode_kernel.cuh -- single-pass VByte decode for sm_100a.
//
// Replaces the reference's Masked-VByte stream loop
// (/root/reference/proj/core/src/stream_loop.hpp:31-129 and the SSE window
// kernels of core/src/decode_simd.cpp:48-148) with one streaming pass over
// HBM.  The reference walks 12-byte windows through a 4096-entry mask table;
// on a GPU the same information -- where every integer ends -- comes straight
// from the continuation bits, and the serial dependency (output index, delta
// prefix) is broken with a single-pass decoupled-lookback scan.
//
// Tile = 256 threads x 16 bytes = 4 KiB of input, taken in ticket order.
//   phase 1  each thread loads its 16 bytes (one 128-bit LDG; neighbours'
//            bytes via warp shuffles) and builds the 16-bit mask of integer
//            ends (terminator bytes: high bit clear), strict-mode error
//            candidates, and V[p] = the 32-bit little-endian concatenation of
//            the 7-bit digits of bytes p..p+4, so an integer starting at s
//            with length L is V[s] & bmsk(7L).  V goes to shared memory.
//   count    popc -> warp/block scan -> the tile's integer count is published
//            at once (decoupled lookback, component 0).
//   scatter  each integer's end position goes to shared memory in tile-local
//            output order (EP[]).
//   phase 2  each thread decodes 8 consecutive integers per pass (values in
//            registers); delta mode scans them (in-thread, warp, block).
//            Warp 0 resolves the tile's first output index by lookback over
//            the predecessors' counts while the other warps decode.
//   delta    the tile's gap sum is published (component 1) and looked back
//            (mod 2^32), giving the carry.
//   store    per-warp transpose through shared memory, then coalesced 32-bit
//            streaming stores (any output alignment).
//   finalize the last CTA to finish turns (total count, first error, end of
//            integer count-1) into the reference's DecodeResult.
//
// The lookback is two-level (tiles, and groups of 32 tiles) with relaxed
// loads: each descriptor is one self-validating 64-bit word (status, launch
// epoch, value), so no acquire/release ordering is needed and descriptors
// never have to be re-zeroed between launches.
//
// Semantics follow the reference oracle decode_scalar/decode_delta_scalar
// (core/src/vbyte.cpp:47-74, internal.hpp:22-37): exactly `count` integers,
// strict mode rejects a 5-byte integer whose fifth byte is >= 0x10 (which
// covers runs of >= 5 continuation bytes), truncation reports the integers
// completed before the fault.  Permissive mode splits a run of continuation
// bytes into 5-byte integers from its start (internal.hpp:36; SURVEY.md §8a
// "cross-path facts"), which needs the position of the last terminator
// before each byte: a third lookback component (max) supplies it.
#pragma once

#include <cassert>
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/mvb_cuda.h"
// Debug builds (-DMVB_CHECKS=1, scripts/r2/gpu_checks.sh): device-side bounds
// assertions on the staging stores, the output ranges and the unit loads (the
// pool's compute-sanitizer is unavailable).
#ifndef MVB_CHECKS
#define MVB_CHECKS 0
#endif
#if MVB_CHECKS
#define MVB_CHECK(c) assert(c)
#else
#define MVB_CHECK(c) ((void)0)
#endif

namespace mvbk {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = 16;                    // input bytes per thread
constexpr int kTile = kThreads * kChunk;      // 4096 input bytes per tile
constexpr int kHalo = 16;                     // local coords: lp = p - tile_pos0 + 16
constexpr int kPasses = 2;                    // phase-2 octet passes: 2 x 256 x 8 >= 4096 ints
constexpr int kEPw = 4 + kTile + 8;           // EPw[3] = previous end, EPw[4 + i] = end of int i (packed)
constexpr int kV = kTile + kHalo;             // V[] words; reused as per-warp transpose buffers
#ifndef MVB_LB_WIDTH
#define MVB_LB_WIDTH 1
#endif
#ifndef MVB_LB_BACKOFF0
#define MVB_LB_BACKOFF0 32
#endif
#ifndef MVB_LB_BACKOFFMAX
#define MVB_LB_BACKOFFMAX 256
#endif
constexpr int kLBWidth = MVB_LB_WIDTH;        // entries per lane per (single-level) lookback round
constexpr int kGroup = 32;                    // tiles per lookback group
#ifndef MVB_LB_WARP
#define MVB_LB_WARP 7
#endif
constexpr int kLBWarp = MVB_LB_WARP;          // warp that runs the lookbacks

constexpr int MODE_STRICT = 0;
constexpr int MODE_PERMISSIVE = 1;

// Tile descriptor status (2 bits) + epoch tag; zeroed memory reads as invalid.
constexpr unsigned long long ST_AGG = 1ull;
constexpr unsigned long long ST_INCL = 2ull;

struct alignas(16) WsHeader {
    unsigned long long ticket;       // next tile / unit to hand out
    unsigned long long done;         // finished-CTA counter
    unsigned long long epoch;        // launches completed on this workspace
    unsigned long long err_idx_inv;  // max(~index) of strict-mode bad integer starts
    unsigned long long err_pos_inv;  // max(~byte position) of the same
    unsigned long long last_end;     // max(position after an integer end), 0 = none
    unsigned long long count_end;    // bytes consumed through integer count-1
    unsigned long long reserved0;
    mvb_result result;               // last result (also copied to res_dev)
    unsigned long long reserved[21];
};
static_assert(sizeof(WsHeader) == 256, "header is 256 bytes");

// Workspace: header | tile descriptors: count [n], sum [n], last-terminator [n]
//            | group descriptors: count [ng], sum [ng] | group accumulators: count [ng], sum [ng]
constexpr int kDescArrays = 3;
constexpr int kGroupArrays = 4;

struct Params {
    const uint8_t* in;         // stream start (any alignment)
    long long mis;             // in - aligned base (0..15)
    long long len;             // bytes scanned: min(in_len, 5*count)
    unsigned long long count;  // integers requested
    uint32_t* out;
    uint32_t prev;
    const uint32_t* prev_dev;  // optional: starting value added from device memory (sharded carry)
    unsigned n_tiles;
    WsHeader* hdr;
    unsigned long long* dcnt;  // per-tile count descriptors
    unsigned long long* dsum;  // per-tile gap-sum descriptors
    unsigned long long* dmax;  // per-tile last-terminator descriptors (permissive)
    unsigned long long* gcnt;  // per-group count descriptors
    unsigned long long* gsum;  // per-group gap-sum descriptors
    unsigned long long* gacc_cnt;  // per-group count accumulators (zeroed by the finalizing CTA)
    unsigned long long* gacc_sum;  // per-group sum accumulators (zeroed by the finalizing CTA)
    unsigned n_groups;
    mvb_result* res_dev;       // optional
    unsigned long long* trace; // optional per-tile timeline (profiling only): 8 x u64 per tile
    int only_if_malformed;     // permissive decode after a strict pass of the same request: run only if that pass
                               // reported a malformed integer (otherwise both modes decode alike and its result stands)
};

// Starting value of the delta scan: the host argument, plus the device-resident
// carry when the caller passes one (written by an earlier kernel on the stream).
__device__ __forceinline__ uint32_t prev_of(const Params& P) {
    return P.prev_dev ? P.prev + *P.prev_dev : P.prev;
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define MVB_TRACE(k)                                                                   \
    do {                                                                               \
        if (P.trace) P.trace[static_cast<unsigned long long>(t) * 8 + (k)] = gtimer(); \
    } while (0)

// ------------------------------------------------------------------ helpers

__device__ __forceinline__ uint4 ldg_stream16(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void stg_stream4(void* p, uint32_t a) {
    asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(a) : "memory");
}

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Mask of `width` low bits, clamped to 32 (bmsk.clamp: width >= 32 -> all ones).
__host__ __device__ __forceinline__ uint32_t bmsk(uint32_t width) {
#ifdef __CUDA_ARCH__
    uint32_t r;
    asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(r) : "r"(width));
    return r;
#else
    return width >= 32 ? 0xFFFFFFFFu : ((1u << width) - 1u);
#endif
}

// bit i = bit 7 of byte i (a 4-lane movemask): one multiply gathers the four
// high bits at bits 28..31 (the other partial products land at bits 7, 14,
// 15, 21, 22, 23 and cannot carry into them).
__host__ __device__ __forceinline__ uint32_t hibits4(uint32_t x) {
    return ((x & 0x80808080u) * 0x204081u) >> 28;
}

// 16-bit movemask of four words (bit 4k+r = bit 7 of byte r of word k).
// Bits 24..27 of each product are zero, so the shifted products need at most
// a mask to drop the stray partial products.
__host__ __device__ __forceinline__ uint32_t hibits16(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3) {
    const uint32_t p0 = (w0 & 0x80808080u) * 0x204081u, p1 = (w1 & 0x80808080u) * 0x204081u;
    const uint32_t p2 = (w2 & 0x80808080u) * 0x204081u, p3 = (w3 & 0x80808080u) * 0x204081u;
    return (p0 >> 28) | (p1 >> 24) | ((p2 >> 20) & 0xF00u) | ((p3 >> 16) & 0xF000u);
}

// 7-bit digits of the four bytes of w, concatenated little-endian (28 bits).
__host__ __device__ __forceinline__ uint32_t digits4(uint32_t w) {
    uint32_t y = (w & 0x007F007Fu) | ((w >> 1) & 0x3F803F80u);
    return (y & 0x3FFFu) | ((y >> 2) & 0x0FFFC000u);
}

// V for the 4 byte positions of word d0 given the next word's digits d1.
__device__ __forceinline__ uint4 vquad(uint32_t d0, uint32_t d1) {
    const uint32_t lo = d0 | (d1 << 28), hi = d1 >> 4;
    return make_uint4(lo, __funnelshift_r(lo, hi, 7), __funnelshift_r(lo, hi, 14), __funnelshift_r(lo, hi, 21));
}

// count/max words: 22-bit epoch, 40-bit value.  sum word: 30-bit epoch, 32-bit value.
template <bool kWide>
__device__ __forceinline__ unsigned long long desc_word(unsigned long long st, unsigned long long epoch,
                                                        unsigned long long v) {
    return kWide ? (st << 62) | ((epoch & 0x3FFFFFFFull) << 32) | (v & 0xFFFFFFFFull)
                 : (st << 62) | ((epoch & 0x3FFFFFull) << 40) | (v & 0xFFFFFFFFFFull);
}

template <bool kWide>
__device__ __forceinline__ unsigned desc_status(unsigned long long w, unsigned long long epoch) {
    const unsigned long long tag = kWide ? ((w >> 32) & 0x3FFFFFFFull) : ((w >> 40) & 0x3FFFFFull);
    const unsigned long long want = kWide ? (epoch & 0x3FFFFFFFull) : (epoch & 0x3FFFFFull);
    return tag == want ? static_cast<unsigned>(w >> 62) : 0u;
}

template <bool kWide>
__device__ __forceinline__ unsigned long long desc_value(unsigned long long w) {
    return kWide ? (w & 0xFFFFFFFFull) : (w & 0xFFFFFFFFFFull);
}

enum LookbackOp { OP_SUM40, OP_SUM32, OP_MAX40 };

template <int Op>
__device__ __forceinline__ unsigned long long lb_combine(unsigned long long a, unsigned long long b) {
    if (Op == OP_MAX40) return a > b ? a : b;
    if (Op == OP_SUM32) return (a + b) & 0xFFFFFFFFull;
    return a + b;
}

// Single-level decoupled lookback by one full warp over descriptor array
// `d`: returns the combination of the aggregates of entries [0, from].  Each
// round examines the 32*kLBWidth nearest unresolved entries; only entries
// nearer than the nearest inclusive prefix must be published, and those are
// re-polled with a short backoff.
template <int Op>
__device__ unsigned long long lookback(const unsigned long long* d, long long from, unsigned long long epoch,
                                       int lane) {
    constexpr bool kWide = (Op == OP_SUM32);
    unsigned long long acc = 0;
    long long base = from;
    while (true) {
        unsigned long long w[kLBWidth];
        unsigned st[kLBWidth];
#pragma unroll
        for (int j = 0; j < kLBWidth; ++j) {
            w[j] = 0;
            st[j] = (base - kLBWidth * lane - j >= 0) ? 0u : static_cast<unsigned>(ST_INCL);
        }
        int first;
        int stop_lane;
        unsigned incl;
        unsigned backoff = MVB_LB_BACKOFF0;
        while (true) {
#pragma unroll
            for (int j = 0; j < kLBWidth; ++j)
                if (st[j] == 0) {
                    w[j] = ld_relaxed(d + (base - kLBWidth * lane - j));
                    st[j] = desc_status<kWide>(w[j], epoch);
                }
            first = kLBWidth;
#pragma unroll
            for (int j = kLBWidth - 1; j >= 0; --j)
                if (st[j] == ST_INCL) first = j;
            incl = __ballot_sync(0xFFFFFFFFu, first < kLBWidth);
            stop_lane = incl ? (__ffs(incl) - 1) : 32;
            bool wait = false;
#pragma unroll
            for (int j = 0; j < kLBWidth; ++j) {
                const bool nearer = lane < stop_lane || (lane == stop_lane && j < first);
                wait = wait || (nearer && st[j] == 0);
            }
            if (!__any_sync(0xFFFFFFFFu, wait)) break;
            if (MVB_LB_BACKOFF0 > 0) {
                __nanosleep(backoff);
                backoff = backoff < MVB_LB_BACKOFFMAX ? backoff * 2 : MVB_LB_BACKOFFMAX;
            }
        }
        unsigned long long v = 0;
#pragma unroll
        for (int j = 0; j < kLBWidth; ++j) {
            const bool take = lane < stop_lane || (lane == stop_lane && j <= first);
            if (take) v = lb_combine<Op>(v, desc_value<kWide>(w[j]));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = lb_combine<Op>(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
        acc = lb_combine<Op>(acc, v);
        if (incl) break;
        base -= 32 * kLBWidth;
    }
    return acc;
}

// Two-level decoupled lookback (sums).  Tiles form groups of kGroup; every
// tile adds its aggregate into its group's accumulator and the last arrival
// publishes the group aggregate; the last tile of a group publishes the group
// inclusive prefix.  A tile first looks at its in-group predecessors (one
// round), and if none is inclusive, looks back over group descriptors (one
// round covers 32 groups = 1024 tiles).  A single-level lookback can only
// advance the inclusive frontier by one window per memory round trip, which
// caps the tile rate far below what HBM sustains.
template <int Op>
__device__ unsigned long long lookback2(const unsigned long long* dtile, const unsigned long long* dgroup,
                                        long long t, unsigned long long epoch, int lane) {
    constexpr bool kWide = (Op == OP_SUM32);
    const long long g = t / kGroup;
    const int k = static_cast<int>(t - g * kGroup);  // in-group index; lanes < k see predecessors
    // Poll in-group predecessors (lane l: tile t-1-l) and the nearest 32
    // groups (lane l: group g-1-l) in the same round trip.
    unsigned long long w = 0, wg = 0;
    unsigned st = 0, sg = (g - 1 - lane >= 0) ? 0u : static_cast<unsigned>(ST_INCL);
    int stop, gstop;
    unsigned incl, gincl;
    unsigned backoff = MVB_LB_BACKOFF0;
    int polls = 0;
    while (true) {
        if (lane < k && st == 0) {
            w = ld_relaxed(dtile + (t - 1 - lane));
            st = desc_status<kWide>(w, epoch);
        }
        if (sg == 0) {
            wg = ld_relaxed(dgroup + (g - 1 - lane));
            sg = desc_status<kWide>(wg, epoch);
        }
        incl = __ballot_sync(0xFFFFFFFFu, lane < k && st == ST_INCL);
        stop = incl ? (__ffs(incl) - 1) : k;  // lanes < stop (and stop itself if inclusive) contribute
        gincl = __ballot_sync(0xFFFFFFFFu, sg == ST_INCL);
        gstop = gincl ? (__ffs(gincl) - 1) : 32;
        const bool wait_tiles = __any_sync(0xFFFFFFFFu, lane < stop && st == 0);
        const bool wait_groups = !incl && g > 0 && __any_sync(0xFFFFFFFFu, lane < gstop && sg == 0);
        if (!wait_tiles && !wait_groups) break;
        if (MVB_LB_BACKOFF0 > 0 && ++polls > 2) {
            __nanosleep(backoff);
            backoff = backoff < MVB_LB_BACKOFFMAX ? backoff * 2 : MVB_LB_BACKOFFMAX;
        }
    }
    unsigned long long v = (lane < stop || (incl && lane == stop)) ? desc_value<kWide>(w) : 0ull;
    if (!incl && g > 0 && (lane < gstop || (gincl && lane == gstop))) v = lb_combine<Op>(v, desc_value<kWide>(wg));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = lb_combine<Op>(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
    if (incl || g == 0 || gincl) return v;
    // more than 32 unresolved groups: continue over older groups
    return lb_combine<Op>(v, lookback<Op>(dgroup, g - 1 - 32, epoch, lane));
}

// Count and gap-sum lookback together (delta mode): both two-level
// descriptor streams are polled in the same round trips.
__device__ void lookback2_cnt_sum(const Params& P, long long t, unsigned long long epoch, int lane,
                                  unsigned long long* cnt_out, uint32_t* sum_out) {
    const long long g = t / kGroup;
    const int k = static_cast<int>(t - g * kGroup);
    unsigned long long wc = 0, ws = 0, wgc = 0, wgs = 0;
    unsigned sc = 0, ss = 0;
    const unsigned g0 = (g - 1 - lane >= 0) ? 0u : static_cast<unsigned>(ST_INCL);
    unsigned sgc = g0, sgs = g0;
    int polls = 0;
    unsigned backoff = MVB_LB_BACKOFF0;
    int stop_c, stop_s, gstop_c, gstop_s;
    unsigned in_c, in_s, gin_c, gin_s;
    while (true) {
        if (lane < k) {
            if (sc == 0) { wc = ld_relaxed(P.dcnt + (t - 1 - lane)); sc = desc_status<false>(wc, epoch); }
            if (ss == 0) { ws = ld_relaxed(P.dsum + (t - 1 - lane)); ss = desc_status<true>(ws, epoch); }
        }
        if (sgc == 0) { wgc = ld_relaxed(P.gcnt + (g - 1 - lane)); sgc = desc_status<false>(wgc, epoch); }
        if (sgs == 0) { wgs = ld_relaxed(P.gsum + (g - 1 - lane)); sgs = desc_status<true>(wgs, epoch); }
        in_c = __ballot_sync(0xFFFFFFFFu, lane < k && sc == ST_INCL);
        in_s = __ballot_sync(0xFFFFFFFFu, lane < k && ss == ST_INCL);
        gin_c = __ballot_sync(0xFFFFFFFFu, sgc == ST_INCL);
        gin_s = __ballot_sync(0xFFFFFFFFu, sgs == ST_INCL);
        stop_c = in_c ? __ffs(in_c) - 1 : k;
        stop_s = in_s ? __ffs(in_s) - 1 : k;
        gstop_c = gin_c ? __ffs(gin_c) - 1 : 32;
        gstop_s = gin_s ? __ffs(gin_s) - 1 : 32;
        bool wait = (lane < stop_c && sc == 0) || (lane < stop_s && ss == 0);
        if (g > 0) wait = wait || (!in_c && lane < gstop_c && sgc == 0) || (!in_s && lane < gstop_s && sgs == 0);
        if (!__any_sync(0xFFFFFFFFu, wait)) break;
        if (MVB_LB_BACKOFF0 > 0 && ++polls > 2) {
            __nanosleep(backoff);
            backoff = backoff < MVB_LB_BACKOFFMAX ? backoff * 2 : MVB_LB_BACKOFFMAX;
        }
    }
    unsigned long long vc = (lane < stop_c || (in_c && lane == stop_c)) ? desc_value<false>(wc) : 0ull;
    unsigned long long vs = (lane < stop_s || (in_s && lane == stop_s)) ? desc_value<true>(ws) : 0ull;
    if (!in_c && g > 0 && (lane < gstop_c || (gin_c && lane == gstop_c))) vc += desc_value<false>(wgc);
    if (!in_s && g > 0 && (lane < gstop_s || (gin_s && lane == gstop_s))) vs += desc_value<true>(wgs);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        vc += __shfl_xor_sync(0xFFFFFFFFu, vc, o);
        vs += __shfl_xor_sync(0xFFFFFFFFu, vs, o);
    }
    if (!in_c && g > 0 && !gin_c) vc += lookback<OP_SUM40>(P.gcnt, g - 1 - 32, epoch, lane);
    if (!in_s && g > 0 && !gin_s) vs += lookback<OP_SUM32>(P.gsum, g - 1 - 32, epoch, lane);
    *cnt_out = vc;
    *sum_out = static_cast<uint32_t>(vs);
}

// Tile aggregate publication for the two-level lookback (one thread).
template <bool kWide>
__device__ __forceinline__ void publish_aggregate(unsigned long long* dtile, unsigned long long* dgroup,
                                                  unsigned long long* gacc, long long t, unsigned n_tiles,
                                                  unsigned long long value, unsigned long long epoch) {
    const long long g = t / kGroup;
    st_relaxed(dtile + t, desc_word<kWide>(t == 0 ? ST_INCL : ST_AGG, epoch, value));
    // accumulator: arrivals in bits 48.., value in the low bits (sums: 32-bit
    // value, carries absorbed by bits 32..47; counts: 40-bit value)
    const unsigned long long old = atomicAdd(gacc + g, (1ull << 48) | value);
    const long long gsize = (static_cast<long long>(n_tiles) - g * kGroup) < kGroup
                                ? static_cast<long long>(n_tiles) - g * kGroup : kGroup;
    if (static_cast<long long>(old >> 48) + 1 == gsize) {
        const unsigned long long total = old + value;
        st_relaxed(dgroup + g, desc_word<kWide>(g == 0 ? ST_INCL : ST_AGG, epoch, total));
    }
}

// After a tile resolved its exclusive prefix `excl`: tile inclusive prefix,
// and the group inclusive prefix when it is the group's last tile.
template <bool kWide>
__device__ __forceinline__ void publish_inclusive(unsigned long long* dtile, unsigned long long* dgroup, long long t,
                                                  unsigned n_tiles, unsigned long long incl_value,
                                                  unsigned long long epoch) {
    st_relaxed(dtile + t, desc_word<kWide>(ST_INCL, epoch, incl_value));
    const long long g = t / kGroup;
    if (t == g * kGroup + kGroup - 1 || t == static_cast<long long>(n_tiles) - 1)
        st_relaxed(dgroup + g, desc_word<kWide>(ST_INCL, epoch, incl_value));
}

// Stream bytes with padding: p < 0 reads as 0x00 (a terminator: the stream
// start is an integer boundary), p >= len reads as 0x80 (no integer ends).
__device__ __forceinline__ uint32_t byte_at(const Params& P, long long p) {
    if (p < 0) return 0x00u;
    if (p >= P.len) return 0x80u;
    return P.in[p];
}

__device__ __forceinline__ uint32_t word_slow(const Params& P, long long p) {
    return byte_at(P, p) | (byte_at(P, p + 1) << 8) | (byte_at(P, p + 2) << 16) | (byte_at(P, p + 3) << 24);
}

// ------------------------------------------------------------------ kernel

__device__ __forceinline__ void stg_stream16(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

// Stores 8 consecutive values per lane (lane l holds the ints at pass offsets
// 8l..8l+7; `out_pass` points at offset 0) as 16-byte-aligned quads.  AH
// (block-uniform) is the number of ints before the first aligned output
// address; the quad that straddles two lanes takes the next lane's first AH
// values by shuffle.  Offsets >= lim are not stored.  The few ints that would
// need a value from another warp are stored singly.
template <int AH>
__device__ __forceinline__ void store_octets(uint32_t* out_pass, const uint32_t (&v)[8], int lane, unsigned lim) {
    uint32_t nx[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) nx[k] = (k < AH) ? __shfl_down_sync(0xFFFFFFFFu, v[k], 1) : 0u;
    const unsigned q = 8u * lane;
    if (AH > 0 && lane == 0) {
#pragma unroll
        for (int k = 0; k < AH; ++k)
            if (static_cast<unsigned>(k) < lim) stg_stream4(out_pass + k, v[k]);
    }
    const unsigned s1 = q + AH;
    if (s1 + 4 <= lim) {
        stg_stream16(out_pass + s1, v[AH], v[AH + 1], v[AH + 2], v[AH + 3]);
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (s1 + k < lim) stg_stream4(out_pass + s1 + k, v[AH + k]);
    }
    const unsigned s2 = s1 + 4;
    uint32_t c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k] = (AH + 4 + k < 8) ? v[(AH + 4 + k) & 7] : nx[(AH + 4 + k - 8) & 3];
    if ((AH == 0 || lane < 31) && s2 + 4 <= lim) {
        stg_stream16(out_pass + s2, c[0], c[1], c[2], c[3]);
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const bool own = AH + 4 + k < 8;
            if (s2 + k < lim && (own || lane < 31)) stg_stream4(out_pass + s2 + k, c[k]);
        }
    }
}

// Shared-memory word at a byte offset from V.
__device__ __forceinline__ uint32_t lds_at(const uint32_t* V, uint32_t byte_off) {
    return *reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(V) + byte_off);
}

// Run by the whole last CTA of a launch once every tile is done: zero the
// group accumulators, turn (total count, first error, end of integer
// count-1) into the reference's DecodeResult, reset the header for the next
// launch and advance the epoch.
__device__ void finalize_launch(const Params& P, unsigned long long epoch, int tid, int nthreads) {
    __threadfence();
    for (unsigned i = tid; i < P.n_groups; i += nthreads) {
        P.gacc_cnt[i] = 0;
        P.gacc_sum[i] = 0;
    }
    if (tid == 0) {
        WsHeader* h = P.hdr;
        const unsigned long long last = ld_relaxed(P.dcnt + (P.n_tiles - 1));
        const unsigned long long total = desc_value<false>(last);
        const unsigned long long err_inv = *reinterpret_cast<volatile unsigned long long*>(&h->err_idx_inv);
        const unsigned long long errpos_inv = *reinterpret_cast<volatile unsigned long long*>(&h->err_pos_inv);
        const unsigned long long last_end = *reinterpret_cast<volatile unsigned long long*>(&h->last_end);
        const unsigned long long count_end = *reinterpret_cast<volatile unsigned long long*>(&h->count_end);
        mvb_result r;
        r.reserved = 0;
        if (err_inv != 0ull && ~err_inv < P.count) {
            r.status = MVB_MALFORMED;
            r.values_written = ~err_inv;
            r.bytes_consumed = ~errpos_inv;
        } else if (total >= P.count) {
            r.status = MVB_OK;
            r.values_written = P.count;
            r.bytes_consumed = count_end;
        } else {
            r.status = MVB_TRUNCATED;
            r.values_written = total;
            r.bytes_consumed = last_end;
        }
        h->result = r;
        if (P.res_dev) *P.res_dev = r;
        h->ticket = 0;
        h->done = 0;
        h->err_idx_inv = 0;
        h->err_pos_inv = 0;
        h->last_end = 0;
        h->count_end = 0;
        h->epoch = epoch;
    }
    __threadfence();
}

template <bool kDelta, int kMode>
__global__ void __launch_bounds__(kThreads, 5) vbyte_decode_kernel(Params P) {
    // V[lp]: digits of bytes lp..lp+4 (local coordinates).  EPw[4 + i] packs
    // the end e_i of tile-local integer i as (4*(e_i+1)) << 16 | 7*(e_i+1):
    // the byte offset in V where the next integer starts, and 7x its position,
    // so that integer i is lds(V, EPw[3+i] >> 16) & bmsk((EPw[4+i] - EPw[3+i]) & 0xFFFF).
    __shared__ __align__(16) uint32_t V[kV];
    __shared__ __align__(16) uint32_t EPw[kEPw];
    __shared__ unsigned s_warp_cnt[kWarps];
    __shared__ uint32_t s_pass_sum[kPasses * kWarps];
    __shared__ long long s_warp_lastT[kWarps];
    __shared__ unsigned long long s_cnt_prefix;
    __shared__ uint32_t s_sum_prefix;
    __shared__ long long s_tile_carryT;
    __shared__ unsigned s_prev_lp;
    __shared__ unsigned s_err;  // (local int index << 16) | (local position of the integer start + 16)
    __shared__ bool s_last;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    // Tiles are handed out by an atomic ticket, not taken from blockIdx: the
    // lookback of tile t waits on tiles < t, and a ticket is only ever held by
    // a running CTA, so every tile waited on is resident whatever order the
    // hardware dispatches CTAs in (finalize_launch resets the ticket).
    __shared__ long long s_tile;
    if (P.only_if_malformed && *reinterpret_cast<volatile int*>(&P.hdr->result.status) != MVB_MALFORMED) return;
    if (threadIdx.x == 0) s_tile = static_cast<long long>(atomicAdd(&P.hdr->ticket, 1ull));
    __syncthreads();
    const long long t = s_tile;
    const unsigned long long epoch = P.hdr->epoch + 1;  // constant during a launch
    if (tid == 0) {
        s_err = 0xFFFFFFFFu;
        MVB_TRACE(0);
    }
    const long long tpos0 = t * kTile - P.mis;  // stream position of the tile's first byte
    const long long p0 = tpos0 + static_cast<long long>(tid) * kChunk;
    const int lp0 = kHalo + tid * kChunk;        // local coordinate of p0

    // ---- loads: own 16 bytes, previous 8 bytes, next 4 bytes ----
    uint32_t w0, w1, w2, w3;
    const bool inside = (p0 >= 0) && (p0 + kChunk <= P.len);
    if (inside) {
        const uint4 q = ldg_stream16(P.in + p0);
        w0 = q.x; w1 = q.y; w2 = q.z; w3 = q.w;
    } else {
        w0 = word_slow(P, p0); w1 = word_slow(P, p0 + 4);
        w2 = word_slow(P, p0 + 8); w3 = word_slow(P, p0 + 12);
    }
    uint32_t wp2 = __shfl_up_sync(0xFFFFFFFFu, w2, 1);
    uint32_t wp3 = __shfl_up_sync(0xFFFFFFFFu, w3, 1);
    uint32_t wn = __shfl_down_sync(0xFFFFFFFFu, w0, 1);
    if (lane == 0) {
        if (p0 - 8 >= 0 && p0 <= P.len) {
            const uint2 q = __ldg(reinterpret_cast<const uint2*>(P.in + p0 - 8));
            wp2 = q.x; wp3 = q.y;
        } else {
            wp2 = word_slow(P, p0 - 8); wp3 = word_slow(P, p0 - 4);
        }
    }
    if (lane == 31) {
        if (p0 + 16 >= 0 && p0 + 20 <= P.len) wn = __ldg(reinterpret_cast<const uint32_t*>(P.in + p0 + 16));
        else wn = word_slow(P, p0 + 16);
    }

    // ---- masks ----
    const uint32_t T16 = hibits16(~w0, ~w1, ~w2, ~w3);  // terminators (high bit clear)
    const uint32_t Tx = (hibits4(~wp2) | (hibits4(~wp3) << 4)) | (T16 << 8) | (hibits4(~wn) << 24);
    const uint32_t Cx = ~Tx & 0x0FFFFFFFu;               // continuation bytes, positions -8..19
    uint32_t inr16 = 0xFFFFu;
    if (!inside) {
        const long long lo = p0 < 0 ? -p0 : 0;
        const long long hi = P.len - p0 < 16 ? P.len - p0 : 16;
        inr16 = (hi <= lo) ? 0u : ((0xFFFFu >> (16 - (hi - lo))) << lo) & 0xFFFFu;
    }

    // ---- integer ends ----
    uint32_t ends16;
    uint32_t bad16 = 0;
    if (kMode == MODE_STRICT) {
        ends16 = T16 & inr16;
        // Integer starts s (predecessor terminates) whose first four bytes are
        // continuation bytes; p = s + 4 is the fifth byte (bit j <-> p = p0 + j).
        const uint32_t five = (Tx >> 3) & (Cx >> 4) & (Cx >> 5) & (Cx >> 6) & (Cx >> 7) & inr16;
        if (five) {
            // fifth byte >= 0x10 (includes a continuation fifth byte) -> malformed
            const uint32_t g0 = w0 | (w0 << 1) | (w0 << 2) | (w0 << 3);
            const uint32_t g1 = w1 | (w1 << 1) | (w1 << 2) | (w1 << 3);
            const uint32_t g2 = w2 | (w2 << 1) | (w2 << 2) | (w2 << 3);
            const uint32_t g3 = w3 | (w3 << 1) | (w3 << 2) | (w3 << 3);
            bad16 = five & hibits16(g0, g1, g2, g3);
        }
        if (tid == 0) {
            const uint32_t tp = Tx & 0xFFu;  // positions -8..-1
            s_prev_lp = (t == 0) ? static_cast<unsigned>(kHalo - 1 + P.mis)  // virtual terminator at -1
                        : tp ? static_cast<unsigned>(8 + 31 - __clz(tp)) : 7u;
        }
    } else {
        // ---- permissive: last terminator before each byte (third lookback) ----
        const long long lastT = T16 ? p0 + (31 - __clz(T16)) : LLONG_MIN;
        long long m = lastT;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xFFFFFFFFu, m, o);
            if (lane >= o && y > m) m = y;
        }
        if (lane == 31) s_warp_lastT[warp] = m;
        long long excl = __shfl_up_sync(0xFFFFFFFFu, m, 1);
        if (lane == 0) excl = LLONG_MIN;
        __syncthreads();
        if (warp == 0) {
            long long tileMax = LLONG_MIN;
#pragma unroll
            for (int k = 0; k < kWarps; ++k) tileMax = s_warp_lastT[k] > tileMax ? s_warp_lastT[k] : tileMax;
            // position + 16 (>= 0: pre-stream padding counts as a terminator); 0 = none
            const unsigned long long aggv = tileMax == LLONG_MIN ? 0ull : static_cast<unsigned long long>(tileMax + 16);
            unsigned long long* d = P.dmax + t;
            if (t == 0) {
                if (lane == 0) {
                    st_relaxed(d, desc_word<false>(ST_INCL, epoch, aggv));
                    s_tile_carryT = -1;  // the virtual terminator before the stream
                }
            } else {
                if (lane == 0) st_relaxed(d, desc_word<false>(ST_AGG, epoch, aggv));
                const unsigned long long c = lookback<OP_MAX40>(P.dmax, t - 1, epoch, lane);
                if (lane == 0) {
                    st_relaxed(d, desc_word<false>(ST_INCL, epoch, c > aggv ? c : aggv));
                    s_tile_carryT = c == 0 ? -1 : static_cast<long long>(c) - 16;
                }
            }
        }
        __syncthreads();
        long long carry = s_tile_carryT;
        for (int k = 0; k < warp; ++k) carry = s_warp_lastT[k] > carry ? s_warp_lastT[k] : carry;
        const long long lt_chunk = excl > carry ? excl : carry;
        // A run of continuation bytes ends an integer at every fifth byte
        // counted from the run start (internal.hpp:36 taken 5 bytes at a time).
        const long long d0 = p0 - lt_chunk;  // run length at p0 if p0 is a continuation byte
        unsigned r = d0 > 0 ? static_cast<unsigned>(d0 % 5) : 1u;
        uint32_t e = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if ((T16 >> j) & 1u) {
                e |= 1u << j;
                r = 1;
            } else {
                if (r == 0) e |= 1u << j;
                r = (r == 4) ? 0 : r + 1;
            }
        }
        ends16 = e & inr16;
        if (tid == 0) {
            // last integer end before the tile: the last terminator, or the
            // last fifth byte of the run that follows it
            if (t == 0) {
                s_prev_lp = static_cast<unsigned>(kHalo - 1 + P.mis);
            } else {
                const long long c = s_tile_carryT;
                const long long end = c + 5 * ((tpos0 - 1 - c) / 5);
                s_prev_lp = static_cast<unsigned>(end - tpos0 + kHalo);
            }
        }
    }

    // ---- block scan of integer counts; publish the tile count at once ----
    const unsigned n_own = __popc(ends16);
    unsigned incl = n_own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp_cnt[warp] = incl;
    __syncthreads();
    unsigned wbase = 0, n_tile = 0;
#pragma unroll
    for (int k = 0; k < kWarps; ++k) {
        const unsigned c = s_warp_cnt[k];
        wbase += (k < warp) ? c : 0u;
        n_tile += c;
    }
    const unsigned tbase = wbase + incl - n_own;  // exclusive prefix of this thread within the tile
    if (tid == 0) {
        MVB_TRACE(1);
        publish_aggregate<false>(P.dcnt, P.gcnt, P.gacc_cnt, t, P.n_tiles, n_tile, epoch);
    }

    // ---- V[p]: digits of bytes p..p+4 ----
    {
        const uint32_t d0 = digits4(w0), d1 = digits4(w1), d2 = digits4(w2), d3 = digits4(w3), dn = digits4(wn);
        uint4* vq = reinterpret_cast<uint4*>(V + lp0);
        vq[0] = vquad(d0, d1);
        vq[1] = vquad(d1, d2);
        vq[2] = vquad(d2, d3);
        vq[3] = vquad(d3, dn);
        if (tid == 0) {  // halo positions -8..-1 (local 8..15)
            const uint32_t dp2 = digits4(wp2), dp3 = digits4(wp3);
            uint4* hq = reinterpret_cast<uint4*>(V + 8);
            hq[0] = vquad(dp2, dp3);
            hq[1] = vquad(dp3, d0);
        }
    }

    // ---- scatter packed end positions (tile-local output order) ----
    {
        constexpr uint32_t kStep = (4u << 16) | 7u;  // one byte position
        const uint32_t x0 = static_cast<uint32_t>(lp0 + 1) * kStep;
        uint32_t* ep = EPw + 4 + tbase;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if ((ends16 >> j) & 1u) {
                *ep = x0 + j * kStep;
                ++ep;
            }
        }
        if (n_own && tbase + n_own == n_tile) {  // zero-width padding for the last octet
            const uint32_t xl = x0 + (31 - __clz(ends16)) * kStep;
#pragma unroll
            for (int k = 0; k < 8; ++k) ep[k] = xl;
        }
        if (kMode == MODE_STRICT && bad16) {
            const int j = __ffs(bad16) - 1;
            const unsigned before = (j >= 4) ? __popc(ends16 & ((1u << (j - 4)) - 1u)) : 0u;
            atomicMin(&s_err, ((tbase + before) << 16) | static_cast<unsigned>(lp0 + j - 4 + 16));
        }
        if (tid == 0) EPw[3] = (s_prev_lp + 1) * kStep;
    }
    __syncthreads();

    // ---- phase 2: 8 consecutive integers per thread per pass ----
    uint32_t val[kPasses][8];
    uint32_t lane_excl[kPasses];  // delta: exclusive prefix of this octet within its warp-pass
#pragma unroll
    for (int p = 0; p < kPasses; ++p) {
        const unsigned u = tid + kThreads * p;
        lane_excl[p] = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) val[p][k] = 0;
        if (kThreads * 8 * p >= n_tile) continue;  // block-uniform
        if (8 * u < n_tile) {
            const uint4 qa = *reinterpret_cast<const uint4*>(EPw + 4 + 8 * u);
            const uint4 qb = *reinterpret_cast<const uint4*>(EPw + 8 + 8 * u);
            const uint32_t xs[9] = {EPw[3 + 8 * u], qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
#pragma unroll
            for (int k = 0; k < 8; ++k)
                val[p][k] = lds_at(V, xs[k] >> 16) & bmsk((xs[k + 1] - xs[k]) & 0xFFFFu);
        }
        if (kDelta) {
#pragma unroll
            for (int k = 1; k < 8; ++k) val[p][k] += val[p][k - 1];
            uint32_t x = val[p][7];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
                if (lane >= o) x += y;
            }
            lane_excl[p] = x - val[p][7];
            if (lane == 31) s_pass_sum[p * kWarps + warp] = x;
        }
    }
    if (tid == 0) MVB_TRACE(3);
    __syncthreads();  // phase 2 done everywhere; counts/sums visible

    // ---- lookbacks (one warp): output index, and for delta the carry ----
    uint32_t wp_base[kPasses] = {0, 0};  // in-tile prefix of this warp-pass (delta)
    uint32_t tile_sum = 0;
    if (kDelta) {
        // prefix over (pass, warp) in output order: lane l holds s_pass_sum[l] for l < 16
        const uint32_t x = (lane < kPasses * kWarps && kThreads * 8 * (lane / kWarps) < n_tile) ? s_pass_sum[lane] : 0u;
        uint32_t sc = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, sc, o);
            if (lane >= o) sc += y;
        }
        tile_sum = __shfl_sync(0xFFFFFFFFu, sc, 31);
#pragma unroll
        for (int p = 0; p < kPasses; ++p) wp_base[p] = __shfl_sync(0xFFFFFFFFu, sc - x, p * kWarps + warp);
    }
    if (warp == kLBWarp) {
        if (kDelta && lane == 0) {
            MVB_TRACE(4);
            publish_aggregate<true>(P.dsum, P.gsum, P.gacc_sum, t, P.n_tiles,
                                    t == 0 ? static_cast<uint32_t>(prev_of(P) + tile_sum) : tile_sum, epoch);
        }
        unsigned long long c = 0;
        uint32_t cs = prev_of(P);
        if (t > 0) {
            if (kDelta) {
                lookback2_cnt_sum(P, t, epoch, lane, &c, &cs);
                if (lane == 0)
                    publish_inclusive<true>(P.dsum, P.gsum, t, P.n_tiles, static_cast<uint32_t>(cs + tile_sum), epoch);
            } else {
                c = lookback2<OP_SUM40>(P.dcnt, P.gcnt, t, epoch, lane);
            }
            if (lane == 0) publish_inclusive<false>(P.dcnt, P.gcnt, t, P.n_tiles, c + n_tile, epoch);
        }
        if (lane == 0) {
            s_cnt_prefix = c;
            s_sum_prefix = cs;
            MVB_TRACE(5);
            // bookkeeping for the DecodeResult
            if (n_tile) {
                const long long e_last = static_cast<long long>(EPw[4 + n_tile - 1] & 0xFFFFu) / 7 - 1;
                atomicMax(&P.hdr->last_end, static_cast<unsigned long long>(tpos0 + e_last - kHalo + 1));
                if (c < P.count && P.count - c <= n_tile) {
                    const unsigned k = static_cast<unsigned>(P.count - c - 1);
                    const long long e_k = static_cast<long long>(EPw[4 + k] & 0xFFFFu) / 7 - 1;
                    P.hdr->count_end = static_cast<unsigned long long>(tpos0 + e_k - kHalo + 1);
                }
            }
            if (kMode == MODE_STRICT && s_err != 0xFFFFFFFFu) {
                const unsigned long long idx = c + (s_err >> 16);
                const long long pos = tpos0 + static_cast<long long>(s_err & 0xFFFFu) - 2 * kHalo;
                if (idx < P.count) {
                    atomicMax(&P.hdr->err_idx_inv, ~idx);
                    atomicMax(&P.hdr->err_pos_inv, ~static_cast<unsigned long long>(pos));
                }
            }
        }
    }
    __syncthreads();

    // ---- store: 16-byte-aligned quads, realigned across lanes by shuffles ----
    {
        const unsigned long long cnt_prefix = s_cnt_prefix;
        const uint32_t carry = kDelta ? s_sum_prefix : 0u;
        const unsigned long long room = P.count > cnt_prefix ? P.count - cnt_prefix : 0ull;
        const unsigned lim = room < n_tile ? static_cast<unsigned>(room) : n_tile;
        const unsigned ah =
            (4u - static_cast<unsigned>(((reinterpret_cast<uintptr_t>(P.out) >> 2) + cnt_prefix) & 3u)) & 3u;
#pragma unroll
        for (int p = 0; p < kPasses; ++p) {
            const unsigned i0 = kThreads * 8 * p + 256 * warp;  // first local int of this warp-pass
            if (i0 >= lim) continue;                              // warp-uniform
            uint32_t v[8];
            const uint32_t b = carry + wp_base[p] + lane_excl[p];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = val[p][k] + b;
            uint32_t* const out_pass = P.out + cnt_prefix + i0;
            const unsigned plim = lim - i0;
            switch (ah) {
                case 0: store_octets<0>(out_pass, v, lane, plim); break;
                case 1: store_octets<1>(out_pass, v, lane, plim); break;
                case 2: store_octets<2>(out_pass, v, lane, plim); break;
                default: store_octets<3>(out_pass, v, lane, plim); break;
            }
        }
    }

    // ---- completion; the last CTA produces the DecodeResult ----
    __syncthreads();
    if (tid == 0) {
        MVB_TRACE(6);
        if (P.trace) {
            unsigned smid;
            asm("mov.u32 %0, %smid;" : "=r"(smid));
            P.trace[static_cast<unsigned long long>(t) * 8 + 7] = (static_cast<unsigned long long>(smid) << 32) | blockIdx.x;
        }
        __threadfence();
        s_last = atomicAdd(&P.hdr->done, 1ull) == P.n_tiles - 1;
    }
    __syncthreads();
    if (!s_last) return;
    finalize_launch(P, epoch, tid, kThreads);
}

// Result for calls that need no decode (count == 0, or empty input).
__global__ void set_result_kernel(mvb_result* res, int status, unsigned long long written,
                                  unsigned long long consumed) {
    mvb_result r;
    r.status = status;
    r.reserved = 0;
    r.values_written = written;
    r.bytes_consumed = consumed;
    *res = r;
}

}  // namespace mvbk
