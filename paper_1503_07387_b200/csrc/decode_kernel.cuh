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
// Tile = 256 threads x 16 bytes = 4 KiB of input.  Per tile:
//   phase 1  each thread loads its 16 bytes (one 128-bit LDG; neighbours'
//            bytes via warp shuffles), builds the 16-bit mask of integer ends
//            (terminator bytes, high bit clear), strict-mode error candidates,
//            and V[p] = the 32-bit little-endian concatenation of the 7-bit
//            digits of bytes p..p+4 (so an integer starting at s with length
//            L is V[s] & bmsk(7L)); V goes to shared memory.
//   scan     popc -> warp/block scan -> tile count; decoupled lookback over
//            per-tile counts gives the tile's first output index.
//   scatter  each integer's end position goes to shared memory in output
//            order (EP[]); group g of 4 outputs is aligned so that its
//            global address is 16-byte aligned.
//   phase 2  warp-contiguous 4-int groups: value = V[e_prev+1] & bmsk(7L);
//            delta mode fuses the prefix sum (warp scan + block scan + a
//            second lookback carry mod 2^32); 128-bit streaming stores.
//   finalize the last CTA to finish turns (total count, first error, end of
//            integer count-1) into the reference's DecodeResult.
//
// Semantics follow the reference oracle decode_scalar/decode_delta_scalar
// (core/src/vbyte.cpp:47-74, internal.hpp:22-37): exactly `count` integers,
// strict mode rejects a 5-byte integer whose fifth byte is >= 0x10 (which
// covers runs of >= 5 continuation bytes), truncation reports the integers
// completed before the fault.  Permissive mode (MODE_PERMISSIVE) splits a run
// of continuation bytes into 5-byte integers from its start (internal.hpp:36;
// SURVEY.md §8a "cross-path facts"), which needs the position of the last
// terminator before each byte: a third lookback component (max) supplies it.
#pragma once

#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/mvb_cuda.h"

namespace mvbk {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = 16;                    // input bytes per thread
constexpr int kTile = kThreads * kChunk;      // 4096 input bytes per tile
constexpr int kHalo = 16;                     // local coords: lp = p - tile_pos0 + 16
constexpr int kMaxGroups = kTile / 4 + 1;     // 4-int output groups per tile (+1 misalignment)
constexpr int kMaxJ = (kMaxGroups + kThreads - 1) / kThreads;  // group slots per lane: 5
constexpr int kEP = kTile + 16;               // end-position slots (u16)
constexpr int kV = kTile + kHalo;             // V[] slots (u32)
constexpr int kDescWords = 4;                 // per tile: count, sum, last-terminator, spare

constexpr int MODE_STRICT = 0;
constexpr int MODE_PERMISSIVE = 1;

// Tile descriptor status (2 bits) + epoch tag; zeroed memory reads as invalid.
constexpr unsigned long long ST_AGG = 1ull;
constexpr unsigned long long ST_INCL = 2ull;

struct alignas(16) WsHeader {
    unsigned long long ticket;       // tile ticket counter
    unsigned long long done;         // finished-CTA counter
    unsigned long long epoch;        // launches completed on this workspace
    unsigned long long err_idx_inv;  // max(~index) of strict-mode bad integer starts
    unsigned long long err_pos_inv;  // max(~byte position) of the same
    unsigned long long last_end;     // max(position after a terminating byte), 0 = none
    unsigned long long count_end;    // bytes consumed through integer count-1
    unsigned long long reserved0;
    mvb_result result;               // last result (also copied to res_dev)
    unsigned long long reserved[21];
};
static_assert(sizeof(WsHeader) == 256, "header is 256 bytes");

struct Params {
    const uint8_t* in;        // stream start (any alignment)
    long long mis;            // in - aligned base (0..15)
    long long len;            // bytes scanned: min(in_len, 5*count)
    unsigned long long count; // integers requested
    uint32_t* out;
    uint32_t prev;
    unsigned n_tiles;
    WsHeader* hdr;
    unsigned long long* desc; // kDescWords * n_tiles
    mvb_result* res_dev;      // optional
};

// ------------------------------------------------------------------ helpers

__device__ __forceinline__ uint4 ldg_stream16(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void stg_stream16(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

__device__ __forceinline__ void stg_stream4(void* p, uint32_t a) {
    asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(a) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
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

// bit i = bit 7 of byte i (a 4-lane movemask).
__host__ __device__ __forceinline__ uint32_t hibits4(uint32_t x) {
    return (((x >> 7) & 0x01010101u) * 0x10204080u) >> 28;
}

// 16-bit movemask of four words (bit 4k+r = bit 7 of byte r of word k).
__host__ __device__ __forceinline__ uint32_t hibits16(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3) {
    // Gather word k's high bits at bit k of each byte, then transpose the
    // 4x4 bit matrix with two delta swaps.
    uint32_t m = ((w0 >> 7) & 0x01010101u) | ((w1 >> 6) & 0x02020202u) |
                 ((w2 >> 5) & 0x04040404u) | ((w3 >> 4) & 0x08080808u);
    // byte r, bit k  ->  want bit 4k + r.  Pack bytes into 16 bits: bit 4r + k.
    m = (m | (m >> 4)) & 0x00FF00FFu;
    m = (m | (m >> 8)) & 0x0000FFFFu;
    // Transpose 4x4 (rows r = nibbles, cols k): swap (r,k) <-> (k,r).
    uint32_t t = (m ^ (m >> 3)) & 0x0A0Au;
    m ^= t ^ (t << 3);
    t = (m ^ (m >> 6)) & 0x00CCu;
    m ^= t ^ (t << 6);
    return m;
}

// 7-bit digits of the four bytes of w, concatenated little-endian (28 bits).
__host__ __device__ __forceinline__ uint32_t digits4(uint32_t w) {
    uint32_t y = (w & 0x007F007Fu) | ((w >> 1) & 0x3F803F80u);
    return (y & 0x3FFFu) | ((y >> 2) & 0x0FFFC000u);
}

__device__ __forceinline__ unsigned long long desc_word(unsigned long long st, unsigned long long epoch,
                                                        unsigned long long v, bool wide_epoch) {
    // count/max words: 22-bit epoch, 40-bit value.  sum word: 30-bit epoch, 32-bit value.
    return wide_epoch ? (st << 62) | ((epoch & 0x3FFFFFFFull) << 32) | (v & 0xFFFFFFFFull)
                      : (st << 62) | ((epoch & 0x3FFFFFull) << 40) | (v & 0xFFFFFFFFFFull);
}

__device__ __forceinline__ unsigned desc_status(unsigned long long w, unsigned long long epoch, bool wide_epoch) {
    const unsigned long long tag = wide_epoch ? ((w >> 32) & 0x3FFFFFFFull) : ((w >> 40) & 0x3FFFFFull);
    const unsigned long long want = wide_epoch ? (epoch & 0x3FFFFFFFull) : (epoch & 0x3FFFFFull);
    return tag == want ? static_cast<unsigned>(w >> 62) : 0u;
}

__device__ __forceinline__ unsigned long long desc_value(unsigned long long w, bool wide_epoch) {
    return wide_epoch ? (w & 0xFFFFFFFFull) : (w & 0xFFFFFFFFFFull);
}

enum LookbackOp { OP_SUM40, OP_SUM32, OP_MAX40 };

template <int Op>
__device__ __forceinline__ unsigned long long lb_combine(unsigned long long a, unsigned long long b) {
    if (Op == OP_MAX40) return a > b ? a : b;
    if (Op == OP_SUM32) return (a + b) & 0xFFFFFFFFull;
    return a + b;
}

// Decoupled lookback by one full warp: returns the combination of the
// aggregates of all tiles < t for descriptor component `comp`.
template <int Op>
__device__ unsigned long long lookback(const unsigned long long* desc, int comp, long long t,
                                       unsigned long long epoch, int lane) {
    constexpr bool wide = (Op == OP_SUM32);
    unsigned long long acc = 0;
    long long base = t - 1;
    while (true) {
        const long long idx = base - lane;
        unsigned long long w = 0;
        unsigned st = ST_INCL;
        bool ready;
        int spins = 0;
        do {
            if (idx >= 0) {
                w = ld_acquire(desc + idx * kDescWords + comp);
                st = desc_status(w, epoch, wide);
            }
            ready = __all_sync(0xFFFFFFFFu, st != 0);
            if (!ready && ++spins > 8) __nanosleep(32);
        } while (!ready);
        const unsigned incl = __ballot_sync(0xFFFFFFFFu, st == ST_INCL);
        const int stop = incl ? (__ffs(incl) - 1) : 31;
        unsigned long long v = (idx >= 0 && lane <= stop) ? desc_value(w, wide) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = lb_combine<Op>(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
        acc = lb_combine<Op>(acc, v);
        if (incl) break;
        base -= 32;
    }
    return acc;
}

// Stream bytes [p, p+4n) with padding: p < 0 reads as 0x00 (a terminator: the
// stream start is an integer boundary), p >= len reads as 0x80 (no integer
// ends there).  Vector load when fully inside.
__device__ __forceinline__ uint32_t byte_at(const Params& P, long long p) {
    if (p < 0) return 0x00u;
    if (p >= P.len) return 0x80u;
    return P.in[p];
}

__device__ __forceinline__ uint32_t word_slow(const Params& P, long long p) {
    return byte_at(P, p) | (byte_at(P, p + 1) << 8) | (byte_at(P, p + 2) << 16) | (byte_at(P, p + 3) << 24);
}

// ------------------------------------------------------------------ kernel

template <bool kDelta, int kMode>
__global__ void __launch_bounds__(kThreads, 4) vbyte_decode_kernel(Params P) {
    __shared__ __align__(16) uint32_t V[kV];
    __shared__ __align__(16) uint16_t EP[kEP];
    __shared__ unsigned long long s_ticket;
    __shared__ unsigned s_warp_cnt[kWarps];
    __shared__ uint32_t s_warp_sum[kWarps];
    __shared__ long long s_warp_lastT[kWarps];
    __shared__ unsigned long long s_cnt_prefix;
    __shared__ uint32_t s_sum_prefix;
    __shared__ long long s_tile_carryT;
    __shared__ unsigned s_prev_lp;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;

    if (tid == 0) s_ticket = atomicAdd(&P.hdr->ticket, 1ull);
    const unsigned long long epoch = P.hdr->epoch + 1;  // read-only during a launch
    __syncthreads();
    const long long t = static_cast<long long>(s_ticket);
    const long long tpos0 = t * kTile - P.mis;          // stream position of the tile's first byte
    const long long p0 = tpos0 + static_cast<long long>(tid) * kChunk;
    const int lp0 = kHalo + tid * kChunk;               // local coordinate of p0

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
    const uint32_t T16 = hibits16(~w0, ~w1, ~w2, ~w3);                  // terminators (high bit clear)
    const uint32_t Tx = (hibits4(~wp2) | (hibits4(~wp3) << 4)) | (T16 << 8) | (hibits4(~wn) << 24);
    const uint32_t Cx = ~Tx & 0x0FFFFFFFu;                               // continuation bytes, positions -8..19
    uint32_t inr16 = 0xFFFFu;
    if (!inside) {
        const long long lo = p0 < 0 ? -p0 : 0;
        const long long hi = P.len - p0 < 16 ? P.len - p0 : 16;
        inr16 = (hi <= lo) ? 0u : ((0xFFFFu >> (16 - (hi - lo))) << lo) & 0xFFFFu;
    }
    // Integer starts s (predecessor terminates) whose first four bytes are
    // continuation bytes; p = s + 4 is the fifth byte (bit j <-> p = p0 + j).
    const uint32_t five = (Tx >> 3) & (Cx >> 4) & (Cx >> 5) & (Cx >> 6) & (Cx >> 7) & inr16;

    // ---- V[p]: digits of bytes p..p+4 ----
    {
        const uint32_t d0 = digits4(w0), d1 = digits4(w1), d2 = digits4(w2), d3 = digits4(w3), dn = digits4(wn);
        uint4* vq = reinterpret_cast<uint4*>(V + lp0);
        uint32_t lo, hi;
        lo = d0 | (d1 << 28); hi = d1 >> 4;
        vq[0] = make_uint4(lo, __funnelshift_r(lo, hi, 7), __funnelshift_r(lo, hi, 14), __funnelshift_r(lo, hi, 21));
        lo = d1 | (d2 << 28); hi = d2 >> 4;
        vq[1] = make_uint4(lo, __funnelshift_r(lo, hi, 7), __funnelshift_r(lo, hi, 14), __funnelshift_r(lo, hi, 21));
        lo = d2 | (d3 << 28); hi = d3 >> 4;
        vq[2] = make_uint4(lo, __funnelshift_r(lo, hi, 7), __funnelshift_r(lo, hi, 14), __funnelshift_r(lo, hi, 21));
        lo = d3 | (dn << 28); hi = dn >> 4;
        vq[3] = make_uint4(lo, __funnelshift_r(lo, hi, 7), __funnelshift_r(lo, hi, 14), __funnelshift_r(lo, hi, 21));
        if (tid == 0) {  // halo positions -8..-1 (local 8..15)
            const uint32_t dp2 = digits4(wp2), dp3 = digits4(wp3);
            uint4* hq = reinterpret_cast<uint4*>(V + 8);
            lo = dp2 | (dp3 << 28); hi = dp3 >> 4;
            hq[0] = make_uint4(lo, __funnelshift_r(lo, hi, 7), __funnelshift_r(lo, hi, 14), __funnelshift_r(lo, hi, 21));
            lo = dp3 | (d0 << 28); hi = d0 >> 4;
            hq[1] = make_uint4(lo, __funnelshift_r(lo, hi, 7), __funnelshift_r(lo, hi, 14), __funnelshift_r(lo, hi, 21));
        }
    }

    // ---- integer ends ----
    uint32_t ends16;
    uint32_t bad16 = 0;
    if (kMode == MODE_STRICT) {
        ends16 = T16 & inr16;
        if (five) {
            // fifth byte >= 0x10 (includes a continuation fifth byte) -> malformed
            const uint32_t g0 = w0 | (w0 << 1) | (w0 << 2) | (w0 << 3);
            const uint32_t g1 = w1 | (w1 << 1) | (w1 << 2) | (w1 << 3);
            const uint32_t g2 = w2 | (w2 << 1) | (w2 << 2) | (w2 << 3);
            const uint32_t g3 = w3 | (w3 << 1) | (w3 << 2) | (w3 << 3);
            bad16 = five & hibits16(g0, g1, g2, g3);
        }
    } else {
        ends16 = 0;  // computed after the last-terminator lookback below
    }

    // ---- permissive: last terminator before each byte (third lookback) ----
    long long lt_chunk = 0;  // position of the last terminator before p0
    if (kMode == MODE_PERMISSIVE) {
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
            // encode position + 16 (>= 0 since pre-stream padding counts as a terminator); 0 = none
            const unsigned long long aggv = tileMax == LLONG_MIN ? 0ull : static_cast<unsigned long long>(tileMax + 16);
            unsigned long long* d = P.desc + t * kDescWords + 2;
            if (t == 0) {
                if (lane == 0) st_release(d, desc_word(ST_INCL, epoch, aggv, false));
                if (lane == 0) s_tile_carryT = -1;  // position -1 is the virtual terminator before the stream
            } else {
                if (lane == 0) st_release(d, desc_word(ST_AGG, epoch, aggv, false));
                const unsigned long long c = lookback<OP_MAX40>(P.desc, 2, t, epoch, lane);
                if (lane == 0) {
                    const unsigned long long incl = c > aggv ? c : aggv;
                    st_release(d, desc_word(ST_INCL, epoch, incl, false));
                    s_tile_carryT = c == 0 ? -1 : static_cast<long long>(c) - 16;
                }
            }
        }
        __syncthreads();
        long long carry = s_tile_carryT;
        for (int k = 0; k < warp; ++k) carry = s_warp_lastT[k] > carry ? s_warp_lastT[k] : carry;
        lt_chunk = excl > carry ? excl : carry;
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
    }

    // ---- block scan of integer counts ----
    const unsigned n_own = __popc(ends16);
    unsigned incl = n_own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp_cnt[warp] = incl;
    // end position (local) of the last integer before the tile
    if (tid == 0) {
        if (kMode == MODE_STRICT) {
            const uint32_t tp = Tx & 0xFFu;  // positions -8..-1
            s_prev_lp = tp ? static_cast<unsigned>(8 + 31 - __clz(tp)) : 7u;
        }
    }
    __syncthreads();
    unsigned wbase = 0, n_tile = 0;
#pragma unroll
    for (int k = 0; k < kWarps; ++k) {
        const unsigned c = s_warp_cnt[k];
        wbase += (k < warp) ? c : 0u;
        n_tile += c;
    }
    const unsigned tbase = wbase + incl - n_own;  // exclusive prefix of this thread within the tile

    if (warp == 0) {
        unsigned long long* d = P.desc + t * kDescWords + 0;
        if (t == 0) {
            if (lane == 0) {
                st_release(d, desc_word(ST_INCL, epoch, n_tile, false));
                s_cnt_prefix = 0;
            }
        } else {
            if (lane == 0) st_release(d, desc_word(ST_AGG, epoch, n_tile, false));
            const unsigned long long c = lookback<OP_SUM40>(P.desc, 0, t, epoch, lane);
            if (lane == 0) {
                st_release(d, desc_word(ST_INCL, epoch, c + n_tile, false));
                s_cnt_prefix = c;
            }
        }
        if (kMode == MODE_PERMISSIVE && lane == 0) {
            // last integer end before the tile: the last terminator, or the
            // last fifth byte of the run that follows it
            const long long c = s_tile_carryT;
            const long long end = c + 5 * ((tpos0 - 1 - c) / 5);
            s_prev_lp = static_cast<unsigned>(end - tpos0 + kHalo);
        }
    }
    if (tid == 0 && t == 0) s_prev_lp = static_cast<unsigned>(kHalo - 1 + P.mis);  // position -1
    __syncthreads();
    const unsigned long long cnt_prefix = s_cnt_prefix;
    const unsigned a_out =
        static_cast<unsigned>((static_cast<unsigned long long>(reinterpret_cast<uintptr_t>(P.out)) >> 2) + cnt_prefix) & 3u;

    // ---- scatter end positions (output order), bookkeeping ----
    {
        unsigned k = tbase;
        uint32_t m = ends16;
        uint16_t* ep = EP + 4 + a_out;
        while (m) {
            const int j = __ffs(m) - 1;
            m &= m - 1;
            ep[k] = static_cast<uint16_t>(lp0 + j);
            if (cnt_prefix + k + 1 == P.count) P.hdr->count_end = static_cast<unsigned long long>(p0 + j + 1);
            ++k;
        }
        if (n_own && k == n_tile) {
            const long long lastp = p0 + (31 - __clz(ends16)) + 1;
            atomicMax(&P.hdr->last_end, static_cast<unsigned long long>(lastp));
        }
        if (kMode == MODE_STRICT && bad16) {
            const int j = __ffs(bad16) - 1;
            const long long s = p0 + j - 4;  // integer start
            const unsigned before = (j >= 4) ? __popc(ends16 & ((1u << (j - 4)) - 1u)) : 0u;
            const unsigned long long idx = cnt_prefix + tbase + before;
            if (idx < P.count) {
                atomicMax(&P.hdr->err_idx_inv, ~idx);
                atomicMax(&P.hdr->err_pos_inv, ~static_cast<unsigned long long>(s));
            }
        }
        if (tid == 0) {
            const uint16_t pv = static_cast<uint16_t>(s_prev_lp);
            for (unsigned q = 0; q <= 3 + a_out; ++q) EP[q] = pv;
        }
        if (tid == 1) {
            const uint16_t pv = static_cast<uint16_t>(s_prev_lp);
            for (unsigned q = 0; q < 4; ++q) EP[4 + a_out + n_tile + q] = pv;
        }
    }
    __syncthreads();

    // ---- phase 2: values, (delta) prefix sum, stores ----
    const unsigned n_groups = n_tile ? (n_tile + a_out + 3) >> 2 : 0u;
    const unsigned gpw = ((n_groups + kThreads - 1) / kThreads) * 32;  // groups per warp
    const unsigned g_begin = warp * gpw;
    uint32_t* const out_base = P.out + cnt_prefix - a_out;  // + 4g is 16-byte aligned
    const long long lim = static_cast<long long>(P.count) - static_cast<long long>(cnt_prefix) + a_out;  // slot < lim stored
    const long long first_slot = a_out;                     // slots [a_out, a_out + n_tile) are real
    const long long end_slot = static_cast<long long>(a_out) + n_tile;

    uint32_t val[kMaxJ][4];
    uint32_t carry = 0;
    uint32_t gexcl[kMaxJ];
#pragma unroll
    for (int jj = 0; jj < kMaxJ; ++jj) {
        const unsigned g = g_begin + 32 * jj + lane;
        val[jj][0] = val[jj][1] = val[jj][2] = val[jj][3] = 0;
        gexcl[jj] = 0;
        if (32u * jj >= gpw) continue;  // warp-uniform
        if (g < n_groups) {
            const uint2 q = *reinterpret_cast<const uint2*>(EP + 4 * g + 4);
            const uint32_t ep = EP[4 * g + 3];
            const uint32_t e0 = q.x & 0xFFFFu, e1 = q.x >> 16, e2 = q.y & 0xFFFFu, e3 = q.y >> 16;
            val[jj][0] = V[ep + 1] & bmsk(7u * (e0 - ep));
            val[jj][1] = V[e0 + 1] & bmsk(7u * (e1 - e0));
            val[jj][2] = V[e1 + 1] & bmsk(7u * (e2 - e1));
            val[jj][3] = V[e2 + 1] & bmsk(7u * (e3 - e2));
            const long long s0 = 4ll * g;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (s0 + k < first_slot || s0 + k >= end_slot) val[jj][k] = 0;
        }
        if (kDelta) {
            // in-group inclusive prefix, then warp scan of group totals
            val[jj][1] += val[jj][0];
            val[jj][2] += val[jj][1];
            val[jj][3] += val[jj][2];
            uint32_t x = val[jj][3];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
                if (lane >= o) x += y;
            }
            gexcl[jj] = carry + x - val[jj][3];
            carry += __shfl_sync(0xFFFFFFFFu, x, 31);
        }
    }

    uint32_t base = 0;
    if (kDelta) {
        if (lane == 0) s_warp_sum[warp] = carry;
        __syncthreads();
        if (warp == 0) {
            uint32_t tile_sum = 0;
#pragma unroll
            for (int k = 0; k < kWarps; ++k) tile_sum += s_warp_sum[k];
            unsigned long long* d = P.desc + t * kDescWords + 1;
            if (t == 0) {
                if (lane == 0) {
                    st_release(d, desc_word(ST_INCL, epoch, P.prev + tile_sum, true));
                    s_sum_prefix = P.prev;
                }
            } else {
                if (lane == 0) st_release(d, desc_word(ST_AGG, epoch, tile_sum, true));
                const uint32_t c = static_cast<uint32_t>(lookback<OP_SUM32>(P.desc, 1, t, epoch, lane));
                if (lane == 0) {
                    st_release(d, desc_word(ST_INCL, epoch, c + tile_sum, true));
                    s_sum_prefix = c;
                }
            }
        }
        __syncthreads();
        base = s_sum_prefix;
#pragma unroll
        for (int k = 0; k < kWarps; ++k) base += (k < warp) ? s_warp_sum[k] : 0u;
    }

#pragma unroll
    for (int jj = 0; jj < kMaxJ; ++jj) {
        const unsigned g = g_begin + 32 * jj + lane;
        if (32u * jj >= gpw) continue;
        if (g >= n_groups) continue;
        uint32_t v0 = val[jj][0], v1 = val[jj][1], v2 = val[jj][2], v3 = val[jj][3];
        if (kDelta) {
            const uint32_t b = base + gexcl[jj];
            v0 += b; v1 += b; v2 += b; v3 += b;
        }
        const long long s0 = 4ll * g;
        uint32_t* dst = out_base + s0;
        if (s0 >= first_slot && s0 + 4 <= end_slot && s0 + 4 <= lim) {
            stg_stream16(dst, v0, v1, v2, v3);
        } else {
            const uint32_t vv[4] = {v0, v1, v2, v3};
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (s0 + k >= first_slot && s0 + k < end_slot && s0 + k < lim) stg_stream4(dst + k, vv[k]);
        }
    }

    // ---- completion; the last CTA produces the DecodeResult ----
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        const unsigned long long d = atomicAdd(&P.hdr->done, 1ull);
        if (d == P.n_tiles - 1) {
            __threadfence();
            WsHeader* h = P.hdr;
            const unsigned long long last = ld_acquire(P.desc + static_cast<unsigned long long>(P.n_tiles - 1) * kDescWords);
            const unsigned long long total = desc_value(last, false);
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
            __threadfence();
        }
    }
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
