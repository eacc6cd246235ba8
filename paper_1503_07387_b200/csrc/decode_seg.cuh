// decode_seg.cuh -- two-kernel strict-mode decoder: segment totals, then one
// warp per segment with its output index and carry known up front.
//
// The stream (in 16-byte-aligned coordinates q = p + mis) is cut into S
// equal segments of a multiple of 512 bytes, about four per resident warp.
//
//   A. vbyte_seg_totals: one warp per segment counts the integers that END
//      in it (terminator bytes) and sums the digit weights of its bytes
//      (digit * 128^(position in its integer), mod 2^32; the sums of the
//      segments before a segment are the value sum of the integers before it
//      plus the partial value of the integer straddling its start, which
//      kernel B subtracts), and rolls both up
//      into per-group (32 segments) accumulators (zero between launches:
//      the finalizing CTA of kernel B re-zeroes them).  It reads the input once;
//      for the SURVEY configs c1/c2/c5 the input then sits in the 126 MB L2
//      for kernel B.
//   B. vbyte_seg_decode: one warp per segment derives the segment's output
//      index and delta carry from the group and segment totals (no lookback,
//      no inter-warp or inter-CTA waiting), then decodes the segment in
//      512-byte slices -- terminator scan, V digit windows and EP end list in
//      warp-private shared memory, phase 2 (8 integers per lane per pass),
//      in-warp delta prefix -- and stores the values directly as
//      16-byte-aligned quads.  The next slice is prefetched into registers
//      while the current one is decoded.
//
// Replaces the reference's stream loop (stream_loop.hpp:31-129) for
// DecodeMode::strict with the semantics of decode_scalar /
// decode_delta_scalar (vbyte.cpp:47-74, internal.hpp:22-37): the DecodeResult
// comes from the first malformed integer, the end of integer count-1, or the
// end of the last integer, recorded in the workspace header by the warps that
// see them and combined by the last CTA.
#pragma once

#include "decode_kernel.cuh"
#include "totals_kernel.cuh"

namespace mvbk {


constexpr int kSegWarps = 4;  // warps per CTA
constexpr int kSegThreads = 32 * kSegWarps;
constexpr int kSegSlice = 512;

struct SegParams {
    const uint8_t* in;  // stream start
    long long mis;      // in - 16-byte-aligned base
    long long len;      // bytes scanned
    unsigned long long count;
    uint32_t* out;
    uint32_t prev;
    const uint32_t* prev_dev;
    long long seg_bytes;  // multiple of 512
    long long n_seg;
    long long n_grp;      // ceil(n_seg / 32)
    unsigned* scnt;       // per-segment integer count
    uint32_t* ssum;       // per-segment value sum mod 2^32
    unsigned long long* gcnt;  // per-group sums of scnt / ssum (zeroed by the finalizing CTA)
    unsigned long long* gsum;
    unsigned long long* ucnt;  // per-supergroup (32 groups) sums of gcnt / gsum (zeroed likewise)
    unsigned long long* usum;
    long long n_sup;           // ceil(n_grp / 32)
    long long a_it0, a_q, a_r; // kernel A: first iteration; iterations per warp (quotient, remainder)
    WsHeader* hdr;
    mvb_result* res_dev;
    // segments [s_lo, s_hi) of this launch pair (the whole stream, or one chunk
    // of a pipelined host decode: group-aligned, chunks launched in order).  The
    // integer count and value sum of the groups before s_lo come from base_in
    // (null: zero); the last CTA of kernel B publishes those before s_hi to
    // base_out (the next chunk's base_in) and chunk_total (host-mapped), and
    // re-zeroes the launch's group accumulators.  Only the final launch
    // produces the DecodeResult and resets the header.
    long long s_lo, s_hi;
    int final_launch;
    const unsigned long long* base_in;         // [count, sum] of the groups before s_lo, or null
    unsigned long long* base_out;              // non-final: [count, sum] of the groups before s_hi
    volatile unsigned long long* chunk_total;  // non-final: integers ending in segments < s_hi
};

// Stream byte at aligned coordinate q (0x00 before the stream: the start is an
// integer boundary; 0x80 after it: no integer ends there).
__device__ __forceinline__ uint32_t seg_byte(const SegParams& S, long long q) {
    const long long p = q - S.mis;
    if (p < 0) return 0x00u;
    if (p >= S.len) return 0x80u;
    return S.in[p];
}
__device__ __forceinline__ uint32_t seg_word(const SegParams& S, long long q) {
    return seg_byte(S, q) | (seg_byte(S, q + 1) << 8) | (seg_byte(S, q + 2) << 16) | (seg_byte(S, q + 3) << 24);
}
__device__ __forceinline__ bool seg_inside(const SegParams& S, long long q, long long n) {
    return q - S.mis >= 0 && q - S.mis + n <= S.len;
}
// 16 bytes at aligned coordinate q (q % 16 == 0)
__device__ __forceinline__ uint4 seg_load16(const SegParams& S, long long q) {
    if (seg_inside(S, q, 16)) return ldg_stream16(S.in - S.mis + q);
    return make_uint4(seg_word(S, q), seg_word(S, q + 4), seg_word(S, q + 8), seg_word(S, q + 12));
}
__device__ __forceinline__ uint32_t seg_inr16(const SegParams& S, long long q0) {
    const long long p0 = q0 - S.mis;
    if (p0 >= 0 && p0 + 16 <= S.len) return 0xFFFFu;
    const long long lo = p0 < 0 ? -p0 : 0;
    const long long hi = S.len - p0 < 16 ? S.len - p0 : 16;
    return (hi <= lo) ? 0u : ((0xFFFFu >> (16 - (hi - lo))) << lo) & 0xFFFFu;
}

// cp.async prefetch of 16 bytes into shared memory (per-thread groups)
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// L2 eviction-priority policies (createpolicy) for cache-hinted accesses
__device__ __forceinline__ unsigned long long l2_evict_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long l2_evict_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// cp.async whose L2 line may go first (the decode's last read of the input)
__device__ __forceinline__ void cp_async16_ef(uint32_t dst, const void* src, unsigned long long pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 x;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "r"(a) : "memory");
    return x;
}

// ------------------------------------------------------------------ kernel A

// Digit-weight sum of one word w (bytes b0..b3) given the 8 preceding bytes
// (p1 = the word before w, p2 = the one before that): every byte's digit
// times 128^(its position within its integer), mod 2^32.  The position is
// read off the high bits of the 1..5 preceding bytes in byte lanes (SWAR):
// position 0 after a terminator, 1 after one continuation byte, ...
// Classes 0/1 weigh 1/128 in one dp4a, 2/3 weigh 2^14/2^21 in a second, 4
// weighs 2^28 in a third (only when `hi`: some byte follows >= 2
// continuation bytes).  `keep` (0x80 per byte) selects the bytes counted.
__device__ __forceinline__ uint32_t word_digit_sum(uint32_t w, uint32_t p1, uint32_t p2, uint32_t keep, bool hi) {
    const uint32_t c1 = __funnelshift_l(p1, w, 8) & 0x80808080u;   // byte before is a continuation byte
    const uint32_t c2 = __funnelshift_l(p1, w, 16) & 0x80808080u;  // 2 before
    const uint32_t b = w & 0x7F7F7F7Fu;
    const uint32_t k0 = ~c1 & keep, k1 = c1 & ~c2 & keep;
    uint32_t s = __dp4a(b, ((k0 >> 7) & 0x01010101u) | (k1 & 0x80808080u), 0u);
    if (hi) {
        const uint32_t c3 = __funnelshift_l(p1, w, 24) & 0x80808080u;
        const uint32_t c4 = p1 & 0x80808080u;
        const uint32_t c5 = __funnelshift_l(p2, p1, 8) & 0x80808080u;
        const uint32_t cc = c1 & c2 & keep;
        const uint32_t k2 = cc & ~c3, k3 = cc & c3 & ~c4, k4 = cc & c3 & c4 & ~c5;
        s += __dp4a(b, ((k2 >> 7) & 0x01010101u) | (k3 & 0x80808080u), 0u) << 14;
        s += __dp4a(b, (k4 >> 7) & 0x01010101u, 0u) << 28;
    }
    return s;
}

// Bytes of word w that follow its last terminator byte (0x80 per byte);
// all four if w has none.
__device__ __forceinline__ uint32_t after_last_terminator(uint32_t w) {
    const uint32_t t = ~w & 0x80808080u;
    if (!t) return 0x80808080u;
    const int hb = 31 - __clz(t);  // bit 7 + 8*i of the last terminator byte i
    return hb >= 31 ? 0u : (0x80808080u << (hb + 1)) & 0x80808080u;
}

#ifndef MVB_HEAD2
#define MVB_HEAD2 1  // range head slices may take the 2-byte path
#endif
#ifndef MVB_A_PDL
#define MVB_A_PDL 1  // delta: kernel A launched as a programmatic dependent of the previous kernel B
#endif
#ifndef MVB_A_MINB
#define MVB_A_MINB 6  // kernel A: minimum resident CTAs per SM (80 registers, no spills; the delta
                      // instantiation took 85 unbounded: 5 CTAs per SM, p50 delta +8%)
#endif
#ifndef MVB_A_CHUNKS
#define MVB_A_CHUNKS 2
#endif
constexpr int kSegAChunks = MVB_A_CHUNKS;          // kernel A: 16-byte chunks per lane per iteration
constexpr int kSegASlice = 512 * kSegAChunks;      // bytes per warp iteration
constexpr int kSegAW = 2 + 4 * kSegAChunks;        // words per lane: 2 halo + the lane's bytes
#ifndef MVB_A_STAGES
#define MVB_A_STAGES 4
#endif
constexpr int kAStages = MVB_A_STAGES;             // kernel A: cp.async ring depth (iterations in flight; a power of 2)
constexpr int kASmem = kSegWarps * kAStages * kSegASlice;

// One warp walks a contiguous run of segments in kSegASlice-byte iterations
// (lane l: 16*kSegAChunks contiguous bytes), prefetching the next iteration across segment
// boundaries.  An integer belongs to the segment holding its terminator: the
// digit sum adds the bytes before a segment that belong to its first integer
// (head, at most 4: lane 0's halo word) and leaves out the bytes after its
// last terminator (tail, at most 4 in canonical data: lane 31's last words).
template <bool kDelta>
__device__ __forceinline__ void seg_totals_run(const SegParams& S, long long s_begin, long long s_end, int lane,
                                               uint32_t ring);

template <bool kDelta>
__global__ void __launch_bounds__(kSegThreads, MVB_A_MINB) vbyte_seg_totals(SegParams S) {
    const int lane = threadIdx.x & 31;
    const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    // balanced runs of kSegASlice-byte iterations (host-computed quotient and
    // remainder: no 64-bit division), independent of the segment boundaries
    const long long it_begin = S.a_it0 + gw * S.a_q + (gw < S.a_r ? gw : S.a_r);
    const long long it_end = it_begin + S.a_q + (gw < S.a_r ? 1 : 0);
    extern __shared__ __align__(128) uint8_t smem_a[];
    const uint32_t ring = static_cast<uint32_t>(__cvta_generic_to_shared(smem_a)) +
                          static_cast<uint32_t>((threadIdx.x >> 5) * kAStages * kSegASlice);
    if (it_begin < it_end) seg_totals_run<kDelta>(S, it_begin, it_end, lane, ring);
    (void)nw;
#if MVB_A_PDL
    // this grid completes only after the preceding grid did (kernel B of the
    // previous decode, or anything else before it in the stream)
    if (kDelta) asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
    // kernel B is launched as a programmatic dependent: it may start (and wait
    // in griddepcontrol.wait) once every CTA of this grid got here
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Digit-weight sums of a lane's words: weight 1 after a terminator, 128
// after one continuation byte -- one funnel shift (the previous byte's high
// bit to bit 0 of each byte) and one IMAD per word, then a dp4a.  Bytes
// after two or more continuation bytes (integers of 3..5 bytes, rare in
// delta-coded lists) also get 128 here; a second pass, taken when any lane of
// the warp has one, corrects them to 2^14 / 2^21 / 2^28.
template <int kW>
__device__ __forceinline__ uint32_t words_digit_sum(const uint32_t (&w)[kW], uint32_t& hi) {
    uint32_t sum = 0;
#pragma unroll
    for (int k = 2; k < kW; ++k) {
        const uint32_t ck = w[k] & 0x80808080u, cp = w[k - 1] & 0x80808080u;
        const uint32_t c1b = __funnelshift_l(cp, ck, 1);  // bit 0 of byte j: byte j-1 continues
        hi |= c1b & __funnelshift_l(cp, ck, 9);          // ... and byte j-2 too
        sum = __dp4a(w[k] & 0x7F7F7F7Fu, c1b * 127u + 0x01010101u, sum);
    }
    return sum;
}
template <int kW>
__device__ __forceinline__ uint32_t words_digit_sum_hi(const uint32_t (&w)[kW]) {
    uint32_t sum = 0;
#pragma unroll
    for (int k = 2; k < kW; ++k) {
        const uint32_t ck = w[k] & 0x80808080u, cp = w[k - 1] & 0x80808080u, cpp = w[k - 2] & 0x80808080u;
        const uint32_t c1 = __funnelshift_l(cp, ck, 8), c2 = __funnelshift_l(cp, ck, 16);
        const uint32_t c3 = __funnelshift_l(cp, ck, 24), c4 = cp;
        const uint32_t c5 = __funnelshift_l(cpp, cp, 8);
        const uint32_t cc = c1 & c2, b = w[k] & 0x7F7F7F7Fu;
        sum += __dp4a(b, ((cc & ~c3) >> 7) | (cc & c3 & ~c4), 0u) << 14;
        sum += __dp4a(b, (cc & c3 & c4 & ~c5) >> 7, 0u) << 28;
        sum -= __dp4a(b, cc >> 7, 0u) << 7;  // the weight 128 the first pass gave them
    }
    return sum;
}

// The weight correction of words_digit_sum_hi when no byte follows three
// continuation bytes (integers of at most 3 bytes, e.g. c4's rare long gaps):
// a byte after exactly two continuation bytes weighs 2^14 instead of the 128
// the first pass gave it.  long4 collects the bytes that follow three (the
// caller then falls back to words_digit_sum_hi).
template <int kW>
__device__ __forceinline__ uint32_t words_digit_sum_hi3(const uint32_t (&w)[kW], uint32_t& long4) {
    uint32_t s = 0;
#pragma unroll
    for (int k = 2; k < kW; ++k) {
        const uint32_t ck = w[k] & 0x80808080u, cp = w[k - 1] & 0x80808080u;
        const uint32_t c1 = __funnelshift_l(cp, ck, 8), c2 = __funnelshift_l(cp, ck, 16);
        const uint32_t c3 = __funnelshift_l(cp, ck, 24);
        const uint32_t cc = c1 & c2;
        long4 |= cc & c3;
        s = __dp4a(w[k] & 0x7F7F7F7Fu, cc >> 7, s);
    }
    return s * (16384u - 128u);
}

template <bool kDelta>
__device__ __forceinline__ void seg_totals_run(const SegParams& S, long long it_begin, long long it_end, int lane,
                                               uint32_t ring) {
    // iterations it_begin .. it_end - 1 of kSegASlice bytes (q = kSegASlice * it);
    // a segment is its_per_seg iterations.  The run's totals go to the segment,
    // group and supergroup accumulators (atomics; zero between launches) each
    // time the run leaves a segment.
    const int its_per_seg = static_cast<int>(S.seg_bytes / kSegASlice);
    const long long q_begin = it_begin * kSegASlice;
    const int n_it = static_cast<int>(it_end - it_begin);
    int i_lo, i_hi;  // iterations whose kSegASlice bytes all lie inside the stream: i_lo <= it < i_hi
    {
        const long long d = S.mis - q_begin, e = S.mis + S.len - q_begin;
        const long long lo = d <= 0 ? 0 : (d + kSegASlice - 1) / kSegASlice;
        const long long hi = e <= 0 ? 0 : e / kSegASlice;
        i_lo = static_cast<int>(lo < n_it ? lo : n_it);
        i_hi = static_cast<int>(hi < n_it ? hi : n_it);
    }
    constexpr int L = 16 * kSegAChunks;  // bytes per lane per iteration
    const uint8_t* const pin = S.in - S.mis + q_begin + L * lane;

    uint32_t pw2 = 0, pw3 = 0;  // the 8 bytes before the current iteration (for lane 0)
    if (lane == 0) {
        if (seg_inside(S, q_begin - 8, 8)) {
            const uint2 v = __ldg(reinterpret_cast<const uint2*>(S.in - S.mis + q_begin - 8));
            pw2 = v.x;
            pw3 = v.y;
        } else {
            pw2 = seg_word(S, q_begin - 8);
            pw3 = seg_word(S, q_begin - 4);
        }
    }
    // interior iterations stream through a kAStages-deep cp.async ring (one
    // commit group per iteration, possibly empty); the others load directly
    const uint32_t rb = ring + L * lane;
#pragma unroll
    for (int j = 0; j < kAStages - 1; ++j) {
        if (j < n_it && j >= i_lo && j < i_hi) {
#pragma unroll
            for (int c = 0; c < kSegAChunks; ++c) cp_async16(rb + kSegASlice * j + 16 * c, pin + kSegASlice * j + 16 * c);
        }
        cp_async_commit();
    }
    bool waited = false;  // griddepcontrol.wait done (MVB_A_PDL)
    uint32_t tcount = 0;  // terminators of the lane's bytes (inside the stream) in the current segment
    uint32_t sum = 0;     // digit-weight sum of the lane's bytes in the current segment
    long long s = it_begin / its_per_seg;
    int to_flush = its_per_seg - static_cast<int>(it_begin - s * its_per_seg);  // iterations left in segment s
    const uint8_t* pf = pin + static_cast<long long>(kSegASlice) * (kAStages - 1);  // prefetch source of it + 3
    uint32_t rd = 0;                                                             // ring offset of iteration it
    for (int it = 0; it < n_it; ++it) {
        {
            const int jn = it + kAStages - 1;
            if (jn >= i_lo && jn < i_hi) {
                const uint32_t d = rb + ((rd + kSegASlice * (kAStages - 1)) & (kSegASlice * kAStages - 1));
#pragma unroll
                for (int c = 0; c < kSegAChunks; ++c) cp_async16(d + 16 * c, pf + 16 * c);
            }
            cp_async_commit();
            pf += kSegASlice;
        }
        const bool inter = it >= i_lo && it < i_hi;  // (warp-uniform)
        uint32_t w[kSegAW];  // w[0], w[1]: the 8 bytes before this lane's bytes; then the lane's words
        uint32_t term = 0;   // edge iterations: terminators inside the stream
        if (inter) {
            cp_async_wait<kAStages - 1>();
#pragma unroll
            for (int c = 0; c < kSegAChunks; ++c) {
                const uint4 x = lds128(rb + rd + 16 * c);
                w[2 + 4 * c] = x.x;
                w[3 + 4 * c] = x.y;
                w[4 + 4 * c] = x.z;
                w[5 + 4 * c] = x.w;
            }
        } else {
            const long long ql = q_begin + static_cast<long long>(kSegASlice) * it + L * lane;
#pragma unroll
            for (int c = 0; c < kSegAChunks; ++c) {
                const uint4 x = seg_load16(S, ql + 16 * c);
                w[2 + 4 * c] = x.x;
                w[3 + 4 * c] = x.y;
                w[4 + 4 * c] = x.z;
                w[5 + 4 * c] = x.w;
                term += __popc(hibits16(~x.x, ~x.y, ~x.z, ~x.w) & seg_inr16(S, ql + 16 * c));
            }
        }
        rd = (rd + kSegASlice) & (kSegASlice * kAStages - 1);
        w[0] = __shfl_up_sync(0xFFFFFFFFu, w[kSegAW - 2], 1);
        w[1] = __shfl_up_sync(0xFFFFFFFFu, w[kSegAW - 1], 1);
        const uint32_t l2 = __shfl_sync(0xFFFFFFFFu, w[kSegAW - 2], 31), l3 = __shfl_sync(0xFFFFFFFFu, w[kSegAW - 1], 31);
        if (lane == 0) {
            w[0] = pw2;
            w[1] = pw3;
        }
        pw2 = l2;
        pw3 = l3;
        // per word, split between the ALU and FMA pipes: ck = continuation bits,
        // c1b = bit 0 of byte j set if byte j-1 continues, weight 1 or 128 per
        // byte (IMAD); the digit-weight sum is dp4a(w, wt) - dp4a(ck, wt) (the
        // high bits weighed in and out again, no 0x7F mask); the continuation
        // bytes accumulate in byte counters
        uint32_t cb = 0, sa = 0, sb = 0;
        uint32_t cp = w[1] & 0x80808080u;
#pragma unroll
        for (int k = 2; k < kSegAW; ++k) {
            const uint32_t ck = w[k] & 0x80808080u;
            const uint32_t c1b = __funnelshift_l(cp, ck, 1);
            const uint32_t wt = c1b * 127u + 0x01010101u;
            sa = __dp4a(w[k], wt, sa);
            sb = __dp4a(ck, wt, sb);
            cb += ck >> 7;
            cp = ck;
        }
        const uint32_t nc = __dp4a(cb, 0x01010101u, 0u);  // continuation bytes of the lane's L bytes
        tcount += inter ? static_cast<uint32_t>(L) - nc : term;
        if (kDelta) {
            sum += sa - sb;
            // sb = 128 x (the weights of the continuation bytes) = 128 x nc unless a
            // continuation byte follows another (bytes 0..31, or bytes -2, -1 in
            // the halo): an integer of 3..5 bytes, whose later bytes need the
            // weights 2^14 / 2^21 / 2^28
            const bool pair = sb != (nc << 7) || ((w[1] & (w[1] << 8)) >> 31);
            if (__any_sync(0xFFFFFFFFu, pair)) {
                uint32_t long4 = 0;
                const uint32_t c3 = words_digit_sum_hi3(w, long4);
                sum += __any_sync(0xFFFFFFFFu, long4 != 0) ? words_digit_sum_hi(w) : c3;
            }
        }
        if (--to_flush == 0 || it + 1 == n_it) {  // leaving segment s: flush
#if MVB_A_PDL
            // (delta) launched as a programmatic dependent of the previous decode's
            // kernel B: its last CTA re-zeroes these accumulators, so the first flush
            // waits for it (the loads and digit sums above overlap its tail)
            if (kDelta && !waited) {
                asm volatile("griddepcontrol.wait;" ::: "memory");
                waited = true;
            }
#endif
            const unsigned c_tot = __reduce_add_sync(0xFFFFFFFFu, tcount);
            const uint32_t s_tot = kDelta ? __reduce_add_sync(0xFFFFFFFFu, sum) : 0u;
            if (lane == 0) {
                atomicAdd(S.scnt + s, c_tot);
                atomicAdd(S.gcnt + (s >> 5), static_cast<unsigned long long>(c_tot));
                atomicAdd(S.ucnt + (s >> 10), static_cast<unsigned long long>(c_tot));
                if (kDelta) {
                    atomicAdd(S.ssum + s, s_tot);
                    atomicAdd(S.gsum + (s >> 5), static_cast<unsigned long long>(s_tot));
                    atomicAdd(S.usum + (s >> 10), static_cast<unsigned long long>(s_tot));
                }
            }
            tcount = 0;
            sum = 0;
            ++s;
            to_flush = its_per_seg;
        }
    }
}

// ------------------------------------------------------------------ kernel B

// A byte range of a buffer in 16-byte-aligned coordinates: byte q lives at
// ab[q]; bytes q < lo read as 0x00 (the range start is an integer boundary),
// bytes q >= hi as 0x80 (no integer ends there).
// x << n with PTX semantics (n >= 32 gives 0)
__device__ __forceinline__ uint32_t shl_clamp(uint32_t x, int n) {
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(n));
    return r;
}
struct ByteRange {
    const uint8_t* ab;
    long long lo, hi;
    long long elo, ehi;  // the caller's buffer (ab coordinates): bytes in [elo, ehi) may be read
};
__device__ __forceinline__ uint32_t r_byte(const ByteRange& R, long long q) {
    if (q < R.lo) return 0x00u;
    if (q >= R.hi) return 0x80u;
    return R.ab[q];
}
__device__ __forceinline__ uint32_t r_word(const ByteRange& R, long long q) {
    return r_byte(R, q) | (r_byte(R, q + 1) << 8) | (r_byte(R, q + 2) << 16) | (r_byte(R, q + 3) << 24);
}
__device__ __forceinline__ bool r_inside(const ByteRange& R, long long q, long long n) { return q >= R.lo && q + n <= R.hi; }
// Byte j of the result: 0xFF if j < n (n <= 0: none, n >= 4: all).
__device__ __forceinline__ uint32_t low_bytes_mask(int n) {
    const int k = n < 0 ? 0 : n > 4 ? 4 : n;
    return ~shl_clamp(0xFFFFFFFFu, 8 * k);
}
// The 16 bytes at q (q a multiple of 16).  A block that straddles the range's
// start or end but lies inside the caller's buffer (a list between its
// neighbours in a batch) is one vector load masked in registers; only a block
// that would touch bytes outside the buffer is assembled byte by byte.
__device__ __forceinline__ uint4 r_load16(const ByteRange& R, long long q) {
    if (r_inside(R, q, 16)) return ldg_stream16(R.ab + q);
    if (q + 16 <= R.lo) return make_uint4(0u, 0u, 0u, 0u);
    if (q >= R.hi) return make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u);
    if (q >= R.elo && q + 16 <= R.ehi) {
        uint4 v = ldg_stream16(R.ab + q);
        // bytes [nl, nh) of the block are inside the range (clamped to +-64)
        const int nl = R.lo - q < -64 ? -64 : static_cast<int>(R.lo - q);
        const int nh = R.hi - q > 64 ? 64 : static_cast<int>(R.hi - q);
        uint32_t* const w = &v.x;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t below = low_bytes_mask(nl - 4 * k);   // bytes before the range: 0x00
            const uint32_t inside = low_bytes_mask(nh - 4 * k);  // bytes past it: 0x80
            (&v.x)[k] = (w[k] & ~below & inside) | (0x80808080u & ~inside);
        }
        return v;
    }
    return make_uint4(r_word(R, q), r_word(R, q + 4), r_word(R, q + 8), r_word(R, q + 12));
}
__device__ __forceinline__ uint32_t r_inr16(const ByteRange& R, long long q0) {
    if (r_inside(R, q0, 16)) return 0xFFFFu;
    const long long lo = R.lo - q0 > 0 ? R.lo - q0 : 0;
    const long long hi = R.hi - q0 < 16 ? R.hi - q0 : 16;
    return (hi <= lo) ? 0u : ((0xFFFFu >> (16 - (hi - lo))) << lo) & 0xFFFFu;
}

// Where a range decode reports what it saw, as it sees it (nothing stays
// live in registers across the slice loop): the first malformed integer
// (output index, range-relative start position) and the end of integer
// limit-1.  Stream decode: the workspace header (atomics, combined by the last
// CTA); batched lists: the warp's own shared-memory slots.
struct RangeSink {
    WsHeader* hdr;                 // stream: non-null
    unsigned long long* err_idx;   // lists: warp slot (init ~0ull)
    long long* err_pos;
    long long* count_end;          // lists: warp slot (init -1)
};
__device__ __forceinline__ void sink_error(const RangeSink& K, unsigned long long idx, long long pos,
                                           unsigned long long limit) {
    if (idx >= limit) return;
    if (K.hdr) {
        atomicMax(&K.hdr->err_idx_inv, ~idx);
        atomicMax(&K.hdr->err_pos_inv, ~static_cast<unsigned long long>(pos));
    } else if (idx < *K.err_idx) {  // one lane, slices in order: no race
        *K.err_idx = idx;
        *K.err_pos = pos;
    }
}
__device__ __forceinline__ void sink_count_end(const RangeSink& K, long long pos) {
    if (K.hdr) K.hdr->count_end = static_cast<unsigned long long>(pos);
    else *K.count_end = pos;
}

// Bits 0..3: which of the 4 bytes before q0 lie before the range end (bytes at
// or past it read as 0x80 and must not count as continuation bytes).
__device__ __forceinline__ uint32_t halo_in_range(const ByteRange& R, long long q0) {
    const long long n = R.hi - (q0 - 4);
    return n >= 4 ? 0xFu : n <= 0 ? 0u : (1u << n) - 1u;
}

// The end of the slice's integer of slice rank r (the lane holding it records
// it): ends = the lane's in-range terminator bits, wexcl / n_own its rank range.
__device__ __forceinline__ void slice_count_end(const ByteRange& R, const RangeSink& K, long long q0, uint32_t ends,
                                                uint32_t r, uint32_t wexcl, uint32_t n_own) {
    if (r < wexcl || r >= wexcl + n_own) return;
    uint32_t m = ends;
    for (uint32_t k = r - wexcl; k > 0; --k) m &= m - 1;
    sink_count_end(K, q0 + (__ffs(m) - 1) + 1 - R.lo);
}

// What a range decode returns (identical in every lane).
struct RangeOut {
    long long last_end;  // -1 if the range holds no integer
    unsigned long long n;
    uint32_t carry;      // delta: the running value after the range's last integer
};

// ------------------------------------------------------------------ lane-local range decode

// The same contract as decode_range, computed the other way round: every lane
// decodes, in registers, the integers whose terminator lies in its own 16
// bytes, and writes them in output order into a warp-private staging buffer;
// the warp then copies the staging buffer out with 16-byte-aligned quads.
//
// Per lane: the 7-bit digits of its words are packed (pack28, 28 bits per
// word) into 56-bit windows (word k-1, word k), so an integer ending at byte t
// of word k is one funnel shift (its end to the top of a register) and one
// shift right by 32 - 7 * length.  The lengths come from a chain over the
// lane's 16 bytes (sh = 32 - 7 * length: 25 after a terminator, 7 less per
// continuation byte), started from the terminators of the 4 bytes before.
// Sixteen static slots, one per byte position; a slot stores iff its byte is
// a terminator.
//
// A slice takes the fast path (lane_slots_fast) when it lies inside the
// range, does not hold integer limit-1 and no lane sees four continuation
// bytes in a row in its 4 bytes before and its own 16 (so every integer has
// 1..4 bytes and none is malformed) -- a warp-uniform test; otherwise the
// general path (ll_slice_gen: range masks, 5-byte integers, malformed
// integers, the end of integer limit-1).  Delta: in-lane running sums stay in
// registers, the warp scan of the lane totals adds the offsets before the
// stores.
#ifndef MVB_FAST5
#define MVB_FAST5 1  // plain slices with canonical 5-byte integers on the fast path
#endif
#ifndef MVB_F5_MIN
#define MVB_F5_MIN 256  // ... when the slice holds at least this many integers (sparser: the general path's per-integer loop)
#endif
#ifndef MVB_GEN_INLINE
#define MVB_GEN_INLINE __noinline__  // the 32-byte-lane general path (rare) as a call
#endif
#ifndef MVB_DELTA32
#define MVB_DELTA32 1  // delta stream decodes on 32-byte lanes too (0: 16-byte lanes, two slices per staging group)
#endif
#ifndef MVB_LL_BLOCKS
#define MVB_LL_BLOCKS 6
#endif
#ifndef MVB_LL_BLOCKS_DELTA
#define MVB_LL_BLOCKS_DELTA 6
#endif
constexpr int kLLBlocks = MVB_LL_BLOCKS;           // resident CTAs per SM the register budget targets (plain)
constexpr int kLLBlocksD = MVB_LL_BLOCKS_DELTA;    // (delta: the running sum and its prefix)
constexpr int kLLSlice = 1024;                     // bytes per slice: 32 lanes x 32 bytes
constexpr int kLaneGroup = 2;                      // (V/EP-sized staging: 2 x 512 integers)
constexpr int kLaneStage = kLaneGroup * 512 + 32;  // staging words per warp (+ alignment), whole 128-byte rows
constexpr int kLLWinBytes = 32 * 72;  // per warp: each lane's eight 8-byte digit windows (72-byte stride: 2 banks apart)
#ifndef MVB_LL_NS
#define MVB_LL_NS 3  // 32-byte-lane input ring: slices (MVB_LL_NS - 1 in flight ahead of the one decoded)
#endif
constexpr int kLLNS = MVB_LL_NS;
constexpr int kLaneWarpBytes = 4 * kLaneStage + kLLNS * kLLSlice;  // staging (+ sparse windows) + input ring
constexpr int kLaneSmem = kSegWarps * kLaneWarpBytes;
static_assert((4 * kLaneStage) % 128 == 0 && kLaneWarpBytes % 128 == 0, "staging rows");

// the sparse plain general path (<= 10 integers per lane: <= 320 per slice,
// staged below 1296 bytes) keeps its digit windows in the top of the staging
// buffer instead
constexpr uint32_t kSparseWin = 4 * kLaneStage - kLLWinBytes;
static_assert(kSparseWin >= 4 * (3 + 320) + 128, "sparse windows above the sparse staging");

// Dense ranges (>= 7/8 integer per byte, i.e. mostly 1-byte integers) swizzle
// the staging addresses: the 16-byte quad index within each 128-byte row is
// XORed with the row index (mod 8).  Their lanes store the integers of a slot
// 16 positions apart -- two banks for the whole warp unswizzled -- while the
// copy-out still reads whole aligned quads.  Other ranges spread their stores
// irregularly over the banks already and keep the plain layout (the swizzle
// costs two ALU instructions per slot).
__device__ __forceinline__ bool range_dense(unsigned long long ints, long long bytes) {
    return bytes > 0 && 8ull * ints >= 7ull * static_cast<unsigned long long>(bytes);
}
template <bool kSwz>
__device__ __forceinline__ uint32_t stg_addr(uint32_t b) { return kSwz ? b ^ ((b >> 3) & 0x70u) : b; }
template <bool kSwz>
__device__ __forceinline__ void sts_stage(uint32_t b, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(stg_addr<kSwz>(b)), "r"(v) : "memory");
}

// 7-bit digits of the four bytes of w, packed LSB first (28 bits).
__device__ __forceinline__ uint32_t pack28(uint32_t w) {
    const uint32_t d = w & 0x7F7F7F7Fu;
    return __dp4a(d, 0x00008001u, 0u) + (__dp4a(d, 0x80010000u, 0u) << 14);
}
// x >> n with PTX semantics (n >= 32, or negative as unsigned, gives 0)
__device__ __forceinline__ uint32_t shr_clamp(uint32_t x, int n) {
    uint32_t r;
    asm("shr.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(n));
    return r;
}

template <bool kDelta>
__device__ __forceinline__ uint32_t lane_scan_offset(uint32_t total, uint32_t& carry) {
    uint32_t xs = total;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, xs, o);
        if ((threadIdx.x & 31) >= o) xs += y;
    }
    const uint32_t ex = carry + xs - total;
    carry += __shfl_sync(0xFFFFFFFFu, xs, 31);
    return ex;
}

// ---- 16-byte lanes (delta decodes): 512-byte slices, two per staging group ----

// Fast slots (see above): sp = shared-memory address of the lane's first
// output.  Per slot e: p = byte e terminates; v = umulhi(top, m) with
// m = 2^(7 * length) (the integer's bits are the top 7 * length bits of top);
// next m = p ? 2^7 : m * 2^7.  The multiplies run on the FMA pipe, leaving the
// (half-rate) ALU pipe the predicate, the selects and the funnel shift.
template <bool kDelta, bool kSwz>
__device__ __forceinline__ void lane_slots_fast16(uint32_t wp3, uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3,
                                                uint32_t T16, uint32_t sp, uint32_t& carry) {
    const uint32_t cm = pack28(wp3), c0 = pack28(w0), c1 = pack28(w1), c2 = pack28(w2), c3 = pack28(w3);
    const uint32_t lo[4] = {cm + (c0 << 28), c0 + (c1 << 28), c1 + (c2 << 28), c2 + (c3 << 28)};
    const uint32_t hi[4] = {c0 >> 4, c1 >> 4, c2 >> 4, c3 >> 4};
    // length of the integer ending at byte 0 = 4 - (last terminator among bytes -4..-1)
    uint32_t m = 1u << (28 - 7 * (31 - __clz(static_cast<int>(hibits4(~wp3)))));
    if (kDelta) {
        // the lane's exclusive prefix up front: digit-weight sum of its 16 bytes,
        // minus its tail (bytes after its last terminator: c3 >> 7 * (t + 1)), plus
        // its head (the same for the 4 bytes before: the previous lane's tail)
        const uint32_t tpl = 31 - __clz(static_cast<int>(hibits4(~wp3)));
        const uint32_t t3 = 31 - __clz(static_cast<int>(T16 >> 12));
        const uint32_t wd[5] = {wp3, w0, w1, w2, w3};
        uint32_t S = 0, hic = 0;
#pragma unroll
        for (int k = 1; k < 5; ++k) {
            const uint32_t ck = wd[k] & 0x80808080u, cp = wd[k - 1] & 0x80808080u;
            const uint32_t c1b = __funnelshift_l(cp, ck, 1);
            hic |= c1b & __funnelshift_l(cp, ck, 9);
            S = __dp4a(wd[k] & 0x7F7F7F7Fu, c1b * 127u + 0x01010101u, S);
        }
        if (__any_sync(0xFFFFFFFFu, hic)) {  // bytes after 2 or 3 continuation bytes: 2^14 / 2^21, not 128
#pragma unroll
            for (int k = 1; k < 5; ++k) {
                const uint32_t ck = wd[k] & 0x80808080u, cp = wd[k - 1] & 0x80808080u;
                const uint32_t c1 = __funnelshift_l(cp, ck, 8), c2 = __funnelshift_l(cp, ck, 16);
                const uint32_t c3 = __funnelshift_l(cp, ck, 24);
                const uint32_t cc = c1 & c2, b = wd[k] & 0x7F7F7F7Fu;
                S += __dp4a(b, ((cc & ~c3) >> 7) | (cc & c3), 0u) << 14;
                S -= __dp4a(b, cc >> 7, 0u) << 7;
            }
        }
        const uint32_t own = S - shr_clamp(c3, 7 * (t3 + 1)) + shr_clamp(cm, 7 * (tpl + 1));
        uint32_t acc = lane_scan_offset<kDelta>(own, carry);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const uint32_t top = __funnelshift_r(lo[e >> 2], hi[e >> 2], 3 + 7 * (e & 3));
#define MVB_SLOT_DELTA(STORE)                                                          \
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"                              \
                 "and.b32 t, %3, %5;\n\t"                                                \
                 "setp.ne.b32 p, t, 0;\n\t"                                              \
                 "mul.hi.u32 t, %4, %2;\n\t"                                             \
                 "@p add.u32 %1, %1, t;\n\t" STORE                                       \
                 "@p add.u32 %0, %0, 4;\n\t"                                             \
                 "mul.lo.u32 t, %2, 128;\n\t"                                            \
                 "selp.b32 %2, 128, t, p;\n\t"                                           \
                 "}"                                                                        \
                 : "+r"(sp), "+r"(acc), "+r"(m)                                             \
                 : "r"(T16), "r"(top), "r"(1u << e)                                         \
                 : "memory")
            if (kSwz)
                MVB_SLOT_DELTA("shr.b32 t, %0, 3;\n\tand.b32 t, t, 0x70;\n\txor.b32 t, t, %0;\n\t"
                               "@p st.shared.u32 [t], %1;\n\t");
            else
                MVB_SLOT_DELTA("@p st.shared.u32 [%0], %1;\n\t");
#undef MVB_SLOT_DELTA
        }
    } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const uint32_t top = __funnelshift_r(lo[e >> 2], hi[e >> 2], 3 + 7 * (e & 3));
#define MVB_SLOT_PLAIN(STORE)                                                          \
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 t, a;\n\t"                           \
                 "and.b32 t, %2, %4;\n\t"                                                \
                 "setp.ne.b32 p, t, 0;\n\t"                                              \
                 "mul.hi.u32 t, %3, %1;\n\t" STORE                                       \
                 "@p add.u32 %0, %0, 4;\n\t"                                             \
                 "mul.lo.u32 t, %1, 128;\n\t"                                            \
                 "selp.b32 %1, 128, t, p;\n\t"                                           \
                 "}"                                                                        \
                 : "+r"(sp), "+r"(m)                                                        \
                 : "r"(T16), "r"(top), "r"(1u << e)                                         \
                 : "memory")
            if (kSwz)
                MVB_SLOT_PLAIN("shr.b32 a, %0, 3;\n\tand.b32 a, a, 0x70;\n\txor.b32 a, a, %0;\n\t"
                               "@p st.shared.u32 [a], t;\n\t");
            else
                MVB_SLOT_PLAIN("@p st.shared.u32 [%0], t;\n\t");
#undef MVB_SLOT_PLAIN
        }
    }
}

// Slots of a slice whose integers all have 1 or 2 bytes (no two consecutive
// continuation bytes in the lane's bytes and the one before them; every
// integer is inside the range): the integer ending at byte t of word k is
//   d(t)                       if byte t-1 is a terminator,
//   d(t-1) | d(t) << 7         if byte t-1 is a continuation byte,
// d = 7-bit digit.  Per word, SWAR builds A (low byte of each candidate:
// d(t), or d(t-1) with bit 0 of d(t) at bit 7) and B (high byte: d(t) >> 1,
// or 0); the candidate of byte t is then one prmt of A and B (bytes 2..3
// replicate the sign of B's byte, which is 0).  Per slot: prmt, the
// terminator predicate, the (running sum and) store, the pointer bump.
// Delta: the lane's integer sum is two dp4a per word over the terminator
// bytes (its integers are complete: an integer straddling into the lane is
// built from the previous lane's last byte), then the warp scan.
// PTX of the 1-2-byte slots (operands: %0 staging pointer, %1 running sum,
// %2 terminator mask, then the A words, then the B words).  One slot: the
// candidate (prmt), the terminator predicate, (the running sum,) the store,
// the pointer bump; S1 swizzles the staging address (see stg_addr).
#define MVB_S2_SLOT_D0S0(A, B, SEL, M) \
    "prmt.b32 v, " A ", " B ", " SEL ";\n\tand.b32 t, %2, " M ";\n\tsetp.ne.b32 p, t, 0;\n\t" \
    "@p st.shared.u32 [%0], v;\n\t@p add.u32 %0, %0, 4;\n\t"
#define MVB_S2_SLOT_D1S0(A, B, SEL, M) \
    "prmt.b32 v, " A ", " B ", " SEL ";\n\tand.b32 t, %2, " M ";\n\tsetp.ne.b32 p, t, 0;\n\t" \
    "@p add.u32 %1, %1, v;\n\t@p st.shared.u32 [%0], %1;\n\t@p add.u32 %0, %0, 4;\n\t"
#define MVB_S2_SLOT_D0S1(A, B, SEL, M) \
    "prmt.b32 v, " A ", " B ", " SEL ";\n\tand.b32 t, %2, " M ";\n\tsetp.ne.b32 p, t, 0;\n\t" \
    "shr.b32 t, %0, 3;\n\tand.b32 t, t, 0x70;\n\txor.b32 t, t, %0;\n\t" \
    "@p st.shared.u32 [t], v;\n\t@p add.u32 %0, %0, 4;\n\t"
#define MVB_S2_SLOT_D1S1(A, B, SEL, M) \
    "prmt.b32 v, " A ", " B ", " SEL ";\n\tand.b32 t, %2, " M ";\n\tsetp.ne.b32 p, t, 0;\n\t" \
    "@p add.u32 %1, %1, v;\n\tshr.b32 t, %0, 3;\n\tand.b32 t, t, 0x70;\n\txor.b32 t, t, %0;\n\t" \
    "@p st.shared.u32 [t], %1;\n\t@p add.u32 %0, %0, 4;\n\t"
#define MVB_S2_WORD(SLOT, A, B, M0, M1, M2, M3) \
    SLOT(A, B, "0xcc40", M0) SLOT(A, B, "0xdd51", M1) SLOT(A, B, "0xee62", M2) SLOT(A, B, "0xff73", M3)
#define MVB_S2_BLOCK4(SLOT)                                                                         \
    "{\n\t.reg .pred p;\n\t.reg .b32 v, t;\n\t"                                                    \
    MVB_S2_WORD(SLOT, "%3", "%7", "0x1", "0x2", "0x4", "0x8")                                       \
    MVB_S2_WORD(SLOT, "%4", "%8", "0x10", "0x20", "0x40", "0x80")                                   \
    MVB_S2_WORD(SLOT, "%5", "%9", "0x100", "0x200", "0x400", "0x800")                               \
    MVB_S2_WORD(SLOT, "%6", "%10", "0x1000", "0x2000", "0x4000", "0x8000") "}"
#define MVB_S2_BLOCK8(SLOT)                                                                         \
    "{\n\t.reg .pred p;\n\t.reg .b32 v, t;\n\t"                                                    \
    MVB_S2_WORD(SLOT, "%3", "%11", "0x1", "0x2", "0x4", "0x8")                                      \
    MVB_S2_WORD(SLOT, "%4", "%12", "0x10", "0x20", "0x40", "0x80")                                  \
    MVB_S2_WORD(SLOT, "%5", "%13", "0x100", "0x200", "0x400", "0x800")                              \
    MVB_S2_WORD(SLOT, "%6", "%14", "0x1000", "0x2000", "0x4000", "0x8000")                          \
    MVB_S2_WORD(SLOT, "%7", "%15", "0x10000", "0x20000", "0x40000", "0x80000")                      \
    MVB_S2_WORD(SLOT, "%8", "%16", "0x100000", "0x200000", "0x400000", "0x800000")                  \
    MVB_S2_WORD(SLOT, "%9", "%17", "0x1000000", "0x2000000", "0x4000000", "0x8000000")              \
    MVB_S2_WORD(SLOT, "%10", "%18", "0x10000000", "0x20000000", "0x40000000", "0x80000000") "}"
#define MVB_S2_OPS4 "r"(A[0]), "r"(A[1]), "r"(A[2]), "r"(A[3]), "r"(B[0]), "r"(B[1]), "r"(B[2]), "r"(B[3])
#define MVB_S2_OPS8                                                                                 \
    "r"(A[0]), "r"(A[1]), "r"(A[2]), "r"(A[3]), "r"(A[4]), "r"(A[5]), "r"(A[6]), "r"(A[7]), "r"(B[0]), \
        "r"(B[1]), "r"(B[2]), "r"(B[3]), "r"(B[4]), "r"(B[5]), "r"(B[6]), "r"(B[7])

__device__ __forceinline__ uint32_t prmt_sign(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}
template <bool kDelta, bool kSwz, int NW>
__device__ __forceinline__ void lane_slots_2b(uint32_t wp3, const uint32_t (&w)[NW], uint32_t T, uint32_t sp,
                                              uint32_t& carry) {
    uint32_t A[NW], B[NW];
    uint32_t own = 0, prev = wp3;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
        const uint32_t P = __funnelshift_l(prev, w[k], 8);  // byte t = byte t-1 of the stream
        const uint32_t cm = prmt_sign(P, 0u, 0xBA98u);  // 0xFF where byte t-1 continues (sign-replicating prmt)
        const uint32_t X = (P & 0x7F7F7F7Fu) | ((w[k] << 7) & 0x80808080u);
        A[k] = (X & cm) | (w[k] & ~cm);
        B[k] = (w[k] >> 1) & 0x3F3F3F3Fu & cm;
        if (kDelta) {
            const uint32_t tm = (~w[k] >> 7) & 0x01010101u;  // terminator bytes
            own = __dp4a(A[k], tm, own);
            own += __dp4a(B[k], tm, 0u) << 8;
        }
        prev = w[k];
    }
    uint32_t acc = 0;
    if (kDelta) acc = lane_scan_offset<kDelta>(own, carry);
    // all 4 * NW slots in one asm block: straight-line predicated code with
    // the pointer and the running sum in fixed registers (separate asm
    // statements per slot made ptxas copy them between slots)
    if constexpr (NW == 4) {
        if (kSwz) {
            if (kDelta) asm volatile(MVB_S2_BLOCK4(MVB_S2_SLOT_D1S1) : "+r"(sp), "+r"(acc) : "r"(T), MVB_S2_OPS4 : "memory");
            else asm volatile(MVB_S2_BLOCK4(MVB_S2_SLOT_D0S1) : "+r"(sp), "+r"(acc) : "r"(T), MVB_S2_OPS4 : "memory");
        } else {
            if (kDelta) asm volatile(MVB_S2_BLOCK4(MVB_S2_SLOT_D1S0) : "+r"(sp), "+r"(acc) : "r"(T), MVB_S2_OPS4 : "memory");
            else asm volatile(MVB_S2_BLOCK4(MVB_S2_SLOT_D0S0) : "+r"(sp), "+r"(acc) : "r"(T), MVB_S2_OPS4 : "memory");
        }
    } else {
        if (kSwz) {
            if (kDelta) asm volatile(MVB_S2_BLOCK8(MVB_S2_SLOT_D1S1) : "+r"(sp), "+r"(acc) : "r"(T), MVB_S2_OPS8 : "memory");
            else asm volatile(MVB_S2_BLOCK8(MVB_S2_SLOT_D0S1) : "+r"(sp), "+r"(acc) : "r"(T), MVB_S2_OPS8 : "memory");
        } else {
            if (kDelta) asm volatile(MVB_S2_BLOCK8(MVB_S2_SLOT_D1S0) : "+r"(sp), "+r"(acc) : "r"(T), MVB_S2_OPS8 : "memory");
            else asm volatile(MVB_S2_BLOCK8(MVB_S2_SLOT_D0S0) : "+r"(sp), "+r"(acc) : "r"(T), MVB_S2_OPS8 : "memory");
        }
    }
}

// General slots: integers of 1..5 bytes, terminators restricted to ends16
// (bytes outside the range), malformed runs decode to garbage (their index
// is reported by ll_slice_gen; nothing after it is meaningful).
template <bool kDelta, bool kSwz>
__device__ __forceinline__ void lane_slots_gen16(uint32_t wp3, uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3,
                                               uint32_t T16, uint32_t ends16, uint32_t sp, uint32_t& carry) {
    const uint32_t cm = pack28(wp3), c0 = pack28(w0), c1 = pack28(w1), c2 = pack28(w2), c3 = pack28(w3);
    const uint32_t lo[4] = {cm + (c0 << 28), c0 + (c1 << 28), c1 + (c2 << 28), c2 + (c3 << 28)};
    const uint32_t hi[4] = {c0 >> 4, c1 >> 4, c2 >> 4, c3 >> 4};
    int sh = 7 * (31 - __clz(static_cast<int>(hibits4(~wp3)))) + 4;  // -3 if no terminator in the 4 bytes before
    uint32_t val[16];
    uint32_t acc = 0;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
        if (e) sh = ((T16 >> (e - 1)) & 1u) ? 25 : sh - 7;
        const int k = e >> 2, t = e & 3;
        const uint32_t top = __funnelshift_r(lo[k], hi[k], 3 + 7 * t);  // packed bits ending with byte e
        uint32_t v = shr_clamp(top, sh);
        if (sh < 0) v = __funnelshift_r(lo[k], hi[k], 7 * t);  // five bytes: the low 32 bits
        if (kDelta) {
            if ((ends16 >> e) & 1u) acc += v;
            val[e] = acc;
        } else if ((ends16 >> e) & 1u) {
            sts_stage<kSwz>(sp, v);
            sp += 4;
        }
    }
    if (kDelta) {
        const uint32_t ex = lane_scan_offset<kDelta>(acc, carry);
#pragma unroll
        for (int e = 0; e < 16; ++e)
            if ((ends16 >> e) & 1u) {
                sts_stage<kSwz>(sp, val[e] + ex);
                sp += 4;
            }
    }
}

// The general path of one slice (after the count scan): malformed integers,
// the end of integer limit-1, then the general slots.
template <bool kDelta, bool kSwz>
__device__ __noinline__ uint32_t ll_slice_gen16(const ByteRange& R, long long q0, uint32_t w0, uint32_t w1, uint32_t w2,
                                          uint32_t w3, uint32_t wp3, uint32_t T16, uint32_t inr16, uint32_t n_own,
                                          uint32_t n_w, uint32_t wexcl, unsigned long long rs,
                                          unsigned long long limit, const RangeSink& K, uint32_t sp,
                                          uint32_t carry) {
    const int lane = threadIdx.x & 31;
    const uint32_t ends16 = T16 & inr16;
    uint32_t wp2 = __shfl_up_sync(0xFFFFFFFFu, w2, 1);
    if (lane == 0) wp2 = r_inside(R, q0 - 8, 4) ? __ldg(reinterpret_cast<const uint32_t*>(R.ab + q0 - 8))
                                                : r_word(R, q0 - 8);
    const uint32_t Tx = hibits4(~wp2) | (hibits4(~wp3) << 4) | (T16 << 8);  // positions -8..15
    const uint32_t Cx = ~Tx & 0x00FFFFFFu;
    const uint32_t run4 = Cx & (Cx >> 1) & (Cx >> 2) & (Cx >> 3);
    uint32_t bad16 = 0;
    if (run4) {  // strict: a fifth byte >= 0x10 (4 continuation bytes after an integer end)
        const uint32_t five = (Tx >> 3) & (run4 >> 4) & inr16;
        if (five) {
            const uint32_t g0 = w0 | (w0 << 1) | (w0 << 2) | (w0 << 3);
            const uint32_t g1 = w1 | (w1 << 1) | (w1 << 2) | (w1 << 3);
            const uint32_t g2 = w2 | (w2 << 1) | (w2 << 2) | (w2 << 3);
            const uint32_t g3 = w3 | (w3 << 1) | (w3 << 2) | (w3 << 3);
            bad16 = five & hibits16(g0, g1, g2, g3);
        }
    }
    if (__any_sync(0xFFFFFFFFu, bad16)) {  // rare: the slice's first malformed integer
        const int j = bad16 ? __ffs(bad16) - 1 : 0;
        unsigned long long idx = bad16 ? rs + wexcl + __popc(ends16 & ((1u << j) - 1u)) : ~0ull;
        long long pos = q0 + j - 4 - R.lo;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long oi = __shfl_xor_sync(0xFFFFFFFFu, idx, o);
            const long long op = __shfl_xor_sync(0xFFFFFFFFu, pos, o);
            if (oi < idx) {
                idx = oi;
                pos = op;
            }
        }
        if (lane == 0) sink_error(K, idx, pos, limit);
    }
    if (n_w == 0) return carry;
    // end of integer limit-1, if it ends in this slice
    if (limit - rs <= n_w && limit - 1 - rs >= wexcl && limit - 1 - rs < wexcl + n_own) {
        uint32_t m = ends16;
        for (unsigned r = static_cast<unsigned>(limit - 1 - rs - wexcl); r > 0; --r) m &= m - 1;
        sink_count_end(K, q0 + (__ffs(m) - 1) + 1 - R.lo);
    }
    lane_slots_gen16<kDelta, kSwz>(wp3, w0, w1, w2, w3, T16, ends16, sp, carry);
    return carry;  // (by value: a noinline function's reference argument lives on the stack)
}

// ---- 32-byte lanes (plain decodes): 1 KiB slices ----

// Fast slots (see above) of a lane's 32 bytes w[0..7]; sp = shared-memory
// address of the lane's first output.  Per slot e: p = byte e terminates;
// v = umulhi(top, m) with m = 2^(7 * length) (the integer's bits are the top
// 7 * length bits of top); next m = p ? 2^7 : m * 2^7.  The multiplies run on
// the FMA pipe, leaving the (half-rate) ALU pipe the predicate, the select
// and the funnel shift.  Delta: the lane's exclusive prefix comes first (SWAR
// digit-weight sum, warp scan), then each slot stores the running sum.
// kF5 (plain only): F5 marks the bytes ending a 5-byte integer (the four bytes
// before continue; the vote has checked that each is a terminator < 0x10).  The
// m chain wraps to 0 there; such a slot takes the window's bits [7t, 7t + 32)
// instead: the four bytes before at bits 0..27, the fifth byte's low 4 bits at
// 28..31 (`decode_scalar`'s acc + (b << 28), internal.hpp:30-36).
template <bool kDelta, bool kSwz, bool kF5 = false>
__device__ __forceinline__ void lane_slots_fast(uint32_t wp3, const uint32_t (&w)[8], uint32_t T32, uint32_t sp,
                                                uint32_t& carry, uint32_t F5 = 0u) {
    const uint32_t tp = hibits4(~wp3);
    const uint32_t cm = pack28(wp3);
    // length of the integer ending at byte 0 = 4 - (last terminator among bytes -4..-1)
    uint32_t m = 1u << (28 - 7 * (31 - __clz(static_cast<int>(tp))));
    uint32_t acc = 0;
    if (kDelta) {
        // digit-weight sum of the 32 bytes, minus the tail (bytes after the last
        // terminator: c7 >> 7 * (t + 1)), plus the head (the same for the 4 bytes
        // before: the previous lane's tail)
        const uint32_t t7 = 31 - __clz(static_cast<int>(T32 >> 28));
        uint32_t S = 0, hic = 0, pv = wp3;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t ck = w[k] & 0x80808080u, cp = pv & 0x80808080u;
            const uint32_t c1b = __funnelshift_l(cp, ck, 1);
            hic |= c1b & __funnelshift_l(cp, ck, 9);
            S = __dp4a(w[k] & 0x7F7F7F7Fu, c1b * 127u + 0x01010101u, S);
            pv = w[k];
        }
        if (__any_sync(0xFFFFFFFFu, hic)) {  // bytes after 2 or 3 continuation bytes: 2^14 / 2^21, not 128
            // first the cheap case (3-byte integers only: one dp4a per word); a
            // byte after three continuation bytes (a 4-byte integer) in any lane
            // takes the full correction
            uint32_t d3 = 0, long4 = 0;
            pv = wp3;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t ck = w[k] & 0x80808080u, cp = pv & 0x80808080u;
                const uint32_t cc = __funnelshift_l(cp, ck, 8) & __funnelshift_l(cp, ck, 16);
                long4 |= cc & __funnelshift_l(cp, ck, 24);
                d3 = __dp4a(w[k] & 0x7F7F7F7Fu, cc >> 7, d3);
                pv = w[k];
            }
            if (!__any_sync(0xFFFFFFFFu, long4 != 0)) {
                S += d3 * (16384u - 128u);
            } else {
                pv = wp3;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t ck = w[k] & 0x80808080u, cp = pv & 0x80808080u;
                    const uint32_t c1 = __funnelshift_l(cp, ck, 8), c2 = __funnelshift_l(cp, ck, 16);
                    const uint32_t c3 = __funnelshift_l(cp, ck, 24);
                    const uint32_t cc = c1 & c2, b = w[k] & 0x7F7F7F7Fu;
                    S += __dp4a(b, ((cc & ~c3) >> 7) | (cc & c3), 0u) << 14;
                    S -= __dp4a(b, cc >> 7, 0u) << 7;
                    pv = w[k];
                }
            }
        }
        const uint32_t own =
            S - shr_clamp(pack28(w[7]), 7 * (t7 + 1)) + shr_clamp(cm, 7 * (32 - __clz(static_cast<int>(tp))));
        acc = lane_scan_offset<kDelta>(own, carry);
    }
    uint32_t cprev = cm;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t ck = pack28(w[k]);
        const uint32_t lo = cprev + (ck << 28), hi = ck >> 4;
        cprev = ck;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int e = 4 * k + t;
            const uint32_t fs = 3 + 7 * t;
            if (kDelta) {
#define MVB_SLOT_DELTA(STORE)                                                          \
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"                              \
                 "and.b32 t, %3, %5;\n\t"                                                \
                 "setp.ne.b32 p, t, 0;\n\t"                                              \
                 "shf.r.wrap.b32 t, %6, %7, %4;\n\t"                                     \
                 "mul.hi.u32 t, t, %2;\n\t"                                              \
                 "@p add.u32 %1, %1, t;\n\t" STORE                                       \
                 "@p add.u32 %0, %0, 4;\n\t"                                             \
                 "mul.lo.u32 t, %2, 128;\n\t"                                            \
                 "selp.b32 %2, 128, t, p;\n\t"                                           \
                 "}"                                                                        \
                 : "+r"(sp), "+r"(acc), "+r"(m)                                             \
                 : "r"(T32), "r"(fs), "r"(1u << e), "r"(lo), "r"(hi)                        \
                 : "memory")
                if (kSwz)
                    MVB_SLOT_DELTA("shr.b32 t, %0, 3;\n\tand.b32 t, t, 0x70;\n\txor.b32 t, t, %0;\n\t"
                                   "@p st.shared.u32 [t], %1;\n\t");
                else
                    MVB_SLOT_DELTA("@p st.shared.u32 [%0], %1;\n\t");
#undef MVB_SLOT_DELTA
            } else {
#define MVB_SLOT_PLAIN5(STORE)                                                         \
    asm volatile("{\n\t.reg .pred p, q;\n\t.reg .b32 t, a;\n\t"                         \
                 "and.b32 t, %2, %4;\n\t"                                                \
                 "setp.ne.b32 p, t, 0;\n\t"                                              \
                 "and.b32 a, %7, %4;\n\t"                                                \
                 "setp.ne.b32 q, a, 0;\n\t"                                              \
                 "shf.r.wrap.b32 t, %5, %6, %3;\n\t"                                     \
                 "mul.hi.u32 t, t, %1;\n\t"                                              \
                 "@q shf.r.wrap.b32 t, %5, %6, %8;\n\t" STORE                            \
                 "@p add.u32 %0, %0, 4;\n\t"                                             \
                 "mul.lo.u32 t, %1, 128;\n\t"                                            \
                 "selp.b32 %1, 128, t, p;\n\t"                                           \
                 "}"                                                                        \
                 : "+r"(sp), "+r"(m)                                                        \
                 : "r"(T32), "r"(fs), "r"(1u << e), "r"(lo), "r"(hi), "r"(F5), "r"(f5s)     \
                 : "memory")
#define MVB_SLOT_PLAIN(STORE)                                                          \
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 t, a;\n\t"                           \
                 "and.b32 t, %2, %4;\n\t"                                                \
                 "setp.ne.b32 p, t, 0;\n\t"                                              \
                 "shf.r.wrap.b32 t, %5, %6, %3;\n\t"                                     \
                 "mul.hi.u32 t, t, %1;\n\t" STORE                                        \
                 "@p add.u32 %0, %0, 4;\n\t"                                             \
                 "mul.lo.u32 t, %1, 128;\n\t"                                            \
                 "selp.b32 %1, 128, t, p;\n\t"                                           \
                 "}"                                                                        \
                 : "+r"(sp), "+r"(m)                                                        \
                 : "r"(T32), "r"(fs), "r"(1u << e), "r"(lo), "r"(hi)                        \
                 : "memory")
                if (kF5) {
                    const uint32_t f5s = 7 * t;
                    if (kSwz)
                        MVB_SLOT_PLAIN5("shr.b32 a, %0, 3;\n\tand.b32 a, a, 0x70;\n\txor.b32 a, a, %0;\n\t"
                                        "@p st.shared.u32 [a], t;\n\t");
                    else
                        MVB_SLOT_PLAIN5("@p st.shared.u32 [%0], t;\n\t");
                } else if (kSwz)
                    MVB_SLOT_PLAIN("shr.b32 a, %0, 3;\n\tand.b32 a, a, 0x70;\n\txor.b32 a, a, %0;\n\t"
                                   "@p st.shared.u32 [a], t;\n\t");
                else
                    MVB_SLOT_PLAIN("@p st.shared.u32 [%0], t;\n\t");
#undef MVB_SLOT_PLAIN
#undef MVB_SLOT_PLAIN5
            }
        }
    }
}

// General slots of one 16-byte half (integers of 1..5 bytes, terminators
// restricted to ends16 = bytes inside the range; malformed runs decode to
// garbage -- their index is reported by ll_slice_gen, nothing after it is
// meaningful).  kMode 0: return the sum of the half's integers; 1: store
// them; 2: store the running sum starting from acc.
template <int kMode, bool kSwz>
__device__ __forceinline__ uint32_t gen_half(uint32_t wp3, uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3,
                                             uint32_t T16, uint32_t ends16, uint32_t sp, uint32_t acc) {
    const uint32_t cm = pack28(wp3), c0 = pack28(w0), c1 = pack28(w1), c2 = pack28(w2), c3 = pack28(w3);
    const uint32_t lo[4] = {cm + (c0 << 28), c0 + (c1 << 28), c1 + (c2 << 28), c2 + (c3 << 28)};
    const uint32_t hi[4] = {c0 >> 4, c1 >> 4, c2 >> 4, c3 >> 4};
    int sh = 7 * (31 - __clz(static_cast<int>(hibits4(~wp3)))) + 4;  // -3 if no terminator in the 4 bytes before
    uint32_t sum = 0;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
        if (e) sh = ((T16 >> (e - 1)) & 1u) ? 25 : sh - 7;
        const int k = e >> 2, t = e & 3;
        const uint32_t top = __funnelshift_r(lo[k], hi[k], 3 + 7 * t);  // packed bits ending with byte e
        uint32_t v = shr_clamp(top, sh);
        if (sh < 0) v = __funnelshift_r(lo[k], hi[k], 7 * t);  // five bytes: the low 32 bits
        if ((ends16 >> e) & 1u) {
            if (kMode == 0) {
                sum += v;
            } else {
                if (kMode == 2) acc += v;
                sts_stage<kSwz>(sp, kMode == 2 ? acc : v);
                sp += 4;
            }
        }
    }
    return sum;
}

// Strict checks of one 16-byte half: the first malformed integer (a fifth byte
// >= 0x10, i.e. 4 continuation bytes after an integer end, then anything but
// 0x00..0x0F) and the end of integer limit-1.
__device__ __forceinline__ void gen_check_half(const ByteRange& R, long long q0, uint32_t w0, uint32_t w1,
                                               uint32_t w2, uint32_t w3, uint32_t wp2, uint32_t wp3, uint32_t T16,
                                               uint32_t inr16, uint32_t n_w, uint32_t wexcl,
                                               unsigned long long rs, unsigned long long limit,
                                               const RangeSink& K) {
    const int lane = threadIdx.x & 31;
    const uint32_t ends16 = T16 & inr16;
    const uint32_t n_own = __popc(ends16);
    const uint32_t Tx = hibits4(~wp2) | (hibits4(~wp3) << 4) | (T16 << 8);  // positions -8..15
    const uint32_t Cx = ~Tx & 0x00FFFFFFu;
    const uint32_t run4 = Cx & (Cx >> 1) & (Cx >> 2) & (Cx >> 3);
    uint32_t bad16 = 0;
    if (run4) {
        const uint32_t five = (Tx >> 3) & (run4 >> 4) & inr16;
        if (five) {
            const uint32_t g0 = w0 | (w0 << 1) | (w0 << 2) | (w0 << 3);
            const uint32_t g1 = w1 | (w1 << 1) | (w1 << 2) | (w1 << 3);
            const uint32_t g2 = w2 | (w2 << 1) | (w2 << 2) | (w2 << 3);
            const uint32_t g3 = w3 | (w3 << 1) | (w3 << 2) | (w3 << 3);
            bad16 = five & hibits16(g0, g1, g2, g3);
        }
    }
    if (__any_sync(0xFFFFFFFFu, bad16)) {  // rare: the half's first malformed integer
        const int j = bad16 ? __ffs(bad16) - 1 : 0;
        unsigned long long idx = bad16 ? rs + wexcl + __popc(ends16 & ((1u << j) - 1u)) : ~0ull;
        long long pos = q0 + j - 4 - R.lo;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long oi = __shfl_xor_sync(0xFFFFFFFFu, idx, o);
            const long long op = __shfl_xor_sync(0xFFFFFFFFu, pos, o);
            if (oi < idx) {
                idx = oi;
                pos = op;
            }
        }
        if (lane == 0) sink_error(K, idx, pos, limit);
    }
    if (n_w && limit - rs <= n_w && limit - 1 - rs >= wexcl && limit - 1 - rs < wexcl + n_own) {
        uint32_t m = ends16;
        for (unsigned r = static_cast<unsigned>(limit - 1 - rs - wexcl); r > 0; --r) m &= m - 1;
        sink_count_end(K, q0 + (__ffs(m) - 1) + 1 - R.lo);
    }
}

// Sparse general slices (plain decodes; few integers per lane, e.g. 5-byte
// ones): instead of 32 static slots, one iteration per integer of the
// busiest lane.  The lane's eight 56-bit digit windows (word k-1, word k) go
// to shared memory; the integer ending at byte e has length 4 - (last
// terminator among bytes e-4..e-1) (5 if none) and is read from window e / 4.
template <bool kSwz>
__device__ __forceinline__ void gen_sparse_plain(uint32_t wp3, const uint4 x0, const uint4 x1, uint32_t T32,
                                                 uint32_t ends32, uint32_t sp, uint32_t win, uint32_t n_iter) {
    const uint32_t w[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
    uint32_t cp = pack28(wp3);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t ck = pack28(w[k]);
        asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(win + 8u * k), "r"(cp + (ck << 28)), "r"(ck >> 4)
                     : "memory");
        cp = ck;
    }
    __syncwarp();
    const uint32_t tlo = hibits4(~wp3) | (T32 << 4), thi = T32 >> 28;  // terminators, positions -4..31
    uint32_t M = ends32;
    for (uint32_t it = 0; it < n_iter; ++it) {
        if (M) {
            const uint32_t e = __ffs(M) - 1;
            M &= M - 1;
            const uint32_t nib = __funnelshift_r(tlo, thi, e) & 0xFu;  // terminators at bytes e-4..e-1
            const uint32_t L = 3u - (31u - __clz(nib)) + 1u;           // 5 if none
            uint2 wd;
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(wd.x), "=r"(wd.y) : "r"(win + 8u * (e >> 2)) : "memory");
            const uint32_t t = e & 3u;
            const uint32_t top = __funnelshift_r(wd.x, wd.y, 3u + 7u * t);  // bits ending with byte e
            const uint32_t v = L >= 5u ? __funnelshift_r(wd.x, wd.y, 7u * t) : __umulhi(top, 1u << (7u * L));
            sts_stage<kSwz>(sp, v);
            sp += 4;
        }
    }
}

// The general path of one slice (lane = 32 bytes w[0..7], as two 16-byte
// halves): strict checks, then the general slots.  Delta: both halves' sums
// first (the output order is lane-major), one warp scan, then the stores.
template <bool kDelta, bool kSwz>
__device__ MVB_GEN_INLINE uint32_t ll_slice_gen(const ByteRange& R, long long q0, const uint4 x0, const uint4 x1,
                                          uint32_t wp2, uint32_t wp3, uint32_t T32, uint32_t inr32, uint32_t n_w,
                                          uint32_t wexcl, unsigned long long rs, unsigned long long limit,
                                          const RangeSink& K, uint32_t sp, uint32_t win, uint32_t carry) {
    const uint32_t e0 = T32 & inr32 & 0xFFFFu, e1 = (T32 & inr32) >> 16;
    gen_check_half(R, q0, x0.x, x0.y, x0.z, x0.w, wp2, wp3, T32 & 0xFFFFu, inr32 & 0xFFFFu, n_w, wexcl, rs, limit,
                   K);
    gen_check_half(R, q0 + 16, x1.x, x1.y, x1.z, x1.w, x0.z, x0.w, T32 >> 16, inr32 >> 16, n_w,
                   wexcl + __popc(e0), rs, limit, K);
    if (n_w == 0) return carry;
    const uint32_t sp1 = sp + 4u * __popc(e0);
    if (kDelta) {
        const uint32_t s0 = gen_half<0, kSwz>(wp3, x0.x, x0.y, x0.z, x0.w, T32 & 0xFFFFu, e0, 0u, 0u);
        const uint32_t s1 = gen_half<0, kSwz>(x0.w, x1.x, x1.y, x1.z, x1.w, T32 >> 16, e1, 0u, 0u);
        const uint32_t ex = lane_scan_offset<kDelta>(s0 + s1, carry);
        gen_half<2, kSwz>(wp3, x0.x, x0.y, x0.z, x0.w, T32 & 0xFFFFu, e0, sp, ex);
        gen_half<2, kSwz>(x0.w, x1.x, x1.y, x1.z, x1.w, T32 >> 16, e1, sp1, ex + s0);
    } else {
        const uint32_t n_iter = __reduce_max_sync(0xFFFFFFFFu, __popc(e0) + __popc(e1));
        if (n_iter <= 10) {  // (at c1 density, 16-20 iterations, the static slots are faster)
            gen_sparse_plain<kSwz>(wp3, x0, x1, T32, T32 & inr32, sp, win, n_iter);
        } else {
            gen_half<1, kSwz>(wp3, x0.x, x0.y, x0.z, x0.w, T32 & 0xFFFFu, e0, sp, 0u);
            gen_half<1, kSwz>(x0.w, x1.x, x1.y, x1.z, x1.w, T32 >> 16, e1, sp1, 0u);
        }
    }
    return carry;
}

// Copy stage[a, a + n) to out[run, run + n), indices below `limit` only;
// stage[i] <-> out[run - a + i] with out + run - a 16-byte aligned.  Whole
// quads in the loop; the partial first quad [a, 4) and last quad
// [end & ~3, end) by lanes 0..3 and 4..7, one integer each.
template <bool kSwz>
__device__ __forceinline__ void stage_out(uint32_t st_base, uint32_t a, uint32_t n, unsigned long long run,
                                          unsigned long long limit, uint32_t* out, int lane) {
    if (run >= limit) return;
    const unsigned long long g0 = run - a;
    const unsigned long long room = limit - g0;
    const uint32_t end = (static_cast<unsigned long long>(a + n) < room) ? a + n : static_cast<uint32_t>(room);
    uint32_t* const ob = out + g0;
    const uint32_t i0 = a ? 4u : 0u, i1 = end & ~3u;
#if MVB_CHECKS
    // every store of this copy-out lies in out[run, min(run + n, limit))
    assert(a < 4u && end <= a + n && g0 + end <= limit && g0 + a == run);
#endif
    {
        // (predicated instructions instead of a branch for lanes 0..7, as stage_out_d3)
        const uint32_t i = lane < 4 ? static_cast<uint32_t>(lane) : i1 + static_cast<uint32_t>(lane - 4);
        const uint32_t p1 = (lane < 8 && (lane < 4 ? (i >= a && i < end && a != 0) : (i < end && i1 >= i0))) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred q1;\n\t.reg .b32 v;\n\tsetp.ne.b32 q1, %0, 0;\n\t"
            "@q1 ld.shared.u32 v, [%1];\n\t@q1 st.global.cs.u32 [%2], v;\n\t}"
            ::"r"(p1), "r"(stg_addr<kSwz>(st_base + 4u * i)), "l"(ob + i)
            : "memory");
    }
    // whole quads: lane l copies quads q = i0/4 + l + 32m.  Swizzled, quad q
    // sits at q ^ ((q >> 3) & 7), and (q >> 3) & 7 only flips bit 2 from one m
    // to the next, so even and odd m each keep one base address advancing by
    // 1 KiB; four quads per iteration with immediate offsets.
    // (the swizzle is a function of the absolute shared-memory address: quad
    // index Q = address / 16)
    uint32_t i = i0 + 4 * lane;
    const uint32_t Q = (st_base >> 4) + (i >> 2);
    const uint32_t Qs = kSwz ? (Q ^ ((Q >> 3) & 7u)) : Q;
    const uint32_t ae = 16u * Qs, ao = kSwz ? 16u * (Qs ^ 4u) : 16u * Qs;
    uint4* dst = reinterpret_cast<uint4*>(ob + i);
    uint32_t off = 0;  // shared-memory bytes advanced (both bases)
    for (; i + 384 < i1; i += 512, off += 2048u, dst += 128) {
        const uint4 v0 = lds128(ae + off), v1 = lds128(ao + off + 512u);
        const uint4 v2 = lds128(ae + off + 1024u), v3 = lds128(ao + off + 1536u);
        __stcs(dst, v0);
        __stcs(dst + 32, v1);
        __stcs(dst + 64, v2);
        __stcs(dst + 96, v3);
    }
    if (i < i1) __stcs(dst, lds128(ae + off));
    if (i + 128 < i1) __stcs(dst + 32, lds128(ao + off + 512u));
    if (i + 256 < i1) __stcs(dst + 64, lds128(ae + off + 1024u));
}

// ---- copy-out by the TMA (plain staging layout only) ----
//
// stage_out's whole quads leave as one bulk copy shared -> global
// (cp.async.bulk, issued by lane 0: no ld.shared / st.global instructions, no
// address arithmetic); the <= 3 + 3 integers of the partial quads at both ends
// by lanes 0..7 as before.  Protocol per staging buffer:
//   writers    st.shared ...; stage_fence() (every lane: its generic-proxy
//              writes become visible to the async proxy); __syncwarp()
//   copy-out   stage_out_bulk() (lane 0 commits one bulk group)
//   next use   stage_wait_read() (lane 0 waits until the TMA has read the
//              buffer); __syncwarp(); st.shared ...
// and stage_wait_all() before the warp's last instruction.
__device__ __forceinline__ void stage_fence() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
#ifndef MVB_WAIT_PRED
#define MVB_WAIT_PRED 1  // stage_wait_read as a predicated instruction instead of a branch (c4 931 -> 917 us)
#endif
__device__ __forceinline__ void stage_wait_read(int lane) {
#if MVB_WAIT_PRED
    asm volatile("{\n\t.reg .pred q;\n\tsetp.eq.s32 q, %0, 0;\n\t@q cp.async.bulk.wait_group.read 0;\n\t}" ::"r"(lane)
                 : "memory");
#else
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#endif
}
__device__ __forceinline__ void stage_wait_all(int lane) {
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void stage_out_bulk(uint32_t st_base, uint32_t a, uint32_t n, unsigned long long run,
                                               unsigned long long limit, uint32_t* out, int lane,
                                               unsigned long long pol) {
    if (run >= limit) return;
    const unsigned long long g0 = run - a;
    const unsigned long long room = limit - g0;
    const uint32_t end = (static_cast<unsigned long long>(a + n) < room) ? a + n : static_cast<uint32_t>(room);
    uint32_t* const ob = out + g0;
    const uint32_t i0 = a ? 4u : 0u, i1 = end & ~3u;
#if MVB_CHECKS
    assert(a < 4u && end <= a + n && g0 + end <= limit && g0 + a == run);
#endif
    // (predicated instructions instead of single-lane branches, as stage_out_d3)
    const uint32_t i = lane < 4 ? static_cast<uint32_t>(lane) : i1 + static_cast<uint32_t>(lane - 4);
    const uint32_t p1 = (lane < 8 && (lane < 4 ? (i >= a && i < end && a != 0) : (i < end && i1 >= i0))) ? 1u : 0u;
    const uint32_t p2 = (lane == 0 && i1 > i0) ? 1u : 0u;
    const uint32_t p3 = lane == 0 ? 1u : 0u;
    asm volatile(
        "{\n\t.reg .pred q1, q2, q3;\n\t.reg .b32 v;\n\t"
        "setp.ne.b32 q1, %0, 0;\n\tsetp.ne.b32 q2, %1, 0;\n\tsetp.ne.b32 q3, %2, 0;\n\t"
        "@q1 ld.shared.u32 v, [%3];\n\t@q1 st.global.cs.u32 [%4], v;\n\t"
        "@q2 cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%5], [%6], %7, %8;\n\t"
        "@q3 cp.async.bulk.commit_group;\n\t}"
        ::"r"(p1), "r"(p2), "r"(p3), "r"(st_base + 4u * i), "l"(ob + i), "l"(ob + i0), "r"(st_base + 4u * i0),
          "r"(4u * (i1 - i0)), "l"(pol)
        : "memory");
}


// ring: shared-memory address of the warp's 2 x kLLSlice-byte input ring.
// Slices (kLLSlice bytes: 32 per lane) are indexed from qs; interior slices
// (inside [R.lo, R.hi)) arrive by cp.async one slice ahead into ring half
// (i & 1), the others are read with range masks.
template <bool kDelta, bool kSwz>
__device__ __forceinline__ void decode_range_ll(const ByteRange& R, long long qs, long long qe,
                                                unsigned long long base, uint32_t carry, unsigned long long limit,
                                                uint32_t* out, uint32_t* stage, uint32_t ring, int lane,
                                                const RangeSink& K, RangeOut& ro) {
    const uint32_t out_w = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(out) >> 2);
    const uint32_t st_base = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
    const int ns = static_cast<int>((qe - qs + kLLSlice - 1) / kLLSlice);
    int i_lo, i_hi;  // interior slices: i_lo <= i < i_hi
    {
        const long long d = R.lo - qs, e = R.hi - qs;
        const long long lo = d <= 0 ? 0 : (d + kLLSlice - 1) / kLLSlice;
        const long long hi = e <= 0 ? 0 : e / kLLSlice;
        i_lo = static_cast<int>(lo < ns ? lo : ns);
        i_hi = static_cast<int>(hi < ns ? hi : ns);
    }
    const uint8_t* const pin = R.ab + qs + 32 * lane;  // this lane's bytes of slice 0
    const uint32_t rbase = ring + 32u * lane;
    unsigned long long run = base;  // output index of the slice's first integer
    int last_i = -1;                // the last slice holding an integer (warp-uniform)
    uint32_t pw2 = 0, pw3 = 0;      // lane 0: the 8 bytes before the slice
    if (lane == 0) {
        if (r_inside(R, qs - 8, 8)) {
            const uint2 v = __ldg(reinterpret_cast<const uint2*>(R.ab + qs - 8));
            pw2 = v.x;
            pw3 = v.y;
        } else {
            pw2 = r_word(R, qs - 8);
            pw3 = r_word(R, qs - 4);
        }
    }
    // input ring of kNS slices, kNS - 1 in flight ahead of the one decoded (one
    // commit group per slice, possibly empty)
    constexpr int kNS = kLLNS;
    const unsigned long long pol = l2_evict_first();
#pragma unroll
    for (int j = 0; j < kNS - 1; ++j) {
        if (j >= i_lo && j < i_hi) {
            cp_async16_ef(rbase + kLLSlice * j, pin + kLLSlice * j, pol);
            cp_async16_ef(rbase + kLLSlice * j + 16, pin + kLLSlice * j + 16, pol);
        }
        cp_async_commit();
    }
    uint32_t o_rd = 0, o_wr = kLLSlice * (kNS - 1);  // ring offsets of slices i and i + kNS - 1
#pragma unroll 1
    for (int i = 0; i < ns; ++i) {
        const uint32_t a = (out_w + static_cast<uint32_t>(run)) & 3u;  // staging offset of the slice
        const bool inter = i >= i_lo && i < i_hi;                      // warp-uniform
        {
            const int j = i + kNS - 1;
            if (j >= i_lo && j < i_hi) {
                cp_async16_ef(rbase + o_wr, pin + static_cast<long long>(kLLSlice) * j, pol);
                cp_async16_ef(rbase + o_wr + 16, pin + static_cast<long long>(kLLSlice) * j + 16, pol);
            }
            cp_async_commit();
            o_wr = o_wr + kLLSlice == kLLSlice * kNS ? 0u : o_wr + kLLSlice;
        }
        const long long q0 = qs + static_cast<long long>(kLLSlice) * i + 32 * lane;
        uint4 x0, x1;
        if (inter) {
            cp_async_wait<kNS - 1>();
            x0 = lds128(rbase + o_rd);
            x1 = lds128(rbase + o_rd + 16);
        } else {
            x0 = r_load16(R, q0);
            x1 = r_load16(R, q0 + 16);
        }
        o_rd = o_rd + kLLSlice == kLLSlice * kNS ? 0u : o_rd + kLLSlice;
        const uint32_t w[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        uint32_t wp3 = __shfl_up_sync(0xFFFFFFFFu, w[7], 1), wp2 = __shfl_up_sync(0xFFFFFFFFu, w[6], 1);
        const uint32_t l3 = __shfl_sync(0xFFFFFFFFu, w[7], 31), l2 = __shfl_sync(0xFFFFFFFFu, w[6], 31);
        if (lane == 0) {
            wp3 = pw3;
            wp2 = pw2;
        }
        pw3 = l3;
        pw2 = l2;
        const uint32_t T32 = hibits16(~w[0], ~w[1], ~w[2], ~w[3]) | (hibits16(~w[4], ~w[5], ~w[6], ~w[7]) << 16);
        const uint32_t inr32 = inter ? 0xFFFFFFFFu : (r_inr16(R, q0) | (r_inr16(R, q0 + 16) << 16));
        const uint32_t n_own = __popc(T32 & inr32);
        uint32_t incl = n_own;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t n_w = __shfl_sync(0xFFFFFFFFu, incl, 31);
        const uint32_t wexcl = incl - n_own;
        // four continuation bytes in a row anywhere in positions -4..31
        // a tail slice (bytes past the range end only, read as 0x80: never
        // terminators) may take the fast paths too (delta: the 2-byte one only --
        // the fast path's lane sum assumes a terminator in the lane's last word);
        // its vote counts continuation bytes inside the range only
        const bool tail = !inter && qs + static_cast<long long>(kLLSlice) * i >= R.lo;
        const unsigned long long C = (static_cast<unsigned long long>(~T32 & inr32) << 4) |
                                     (~hibits4(~wp3) & (inter ? 0xFu : halo_in_range(R, q0)));
        const unsigned long long pair = C & (C >> 1);                       // bit j: positions j-4, j-3 continue
        const unsigned long long run2 = pair & 0xFFFFFFFFCull;              // a 3+-byte integer ends in 0..31
        const unsigned long long run4 = pair & (pair >> 2) & 0x1FFFFFFFFull;  // a 5+-byte integer ends in 0..31
        const unsigned vote = (__any_sync(0xFFFFFFFFu, run2 != 0) ? 1u : 0u) | (__any_sync(0xFFFFFFFFu, run4 != 0) ? 2u : 0u);
        // (a head slice -- bytes before the range start, read as 0x00 -- may take
        // the 2-byte path too: its slots store at in-range terminators only, and
        // the zero bytes add nothing to the candidates or the lane sums)
        const bool take2 = (inter || tail || MVB_HEAD2) && vote == 0;
        const bool takef = !take2 && (inter || (tail && !kDelta)) && !(vote & 2u);
        // plain decode: 5-byte integers stay on the fast path (in slices dense
        // enough for 32 slots to pay) when every byte
        // after four continuation bytes (inside the range) is a terminator < 0x10
        // (strict mode's check; longer runs then cannot occur either)
        uint32_t F5 = 0u;
        bool takef5 = false;
        if (!kDelta && MVB_FAST5 && (vote & 2u) && (inter || tail) && n_w >= MVB_F5_MIN) {
            uint32_t y[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) y[k] = w[k] | (w[k] << 1) | (w[k] << 2) | (w[k] << 3);
            const uint32_t nz = hibits16(y[0], y[1], y[2], y[3]) | (hibits16(y[4], y[5], y[6], y[7]) << 16);
            F5 = static_cast<uint32_t>(run4) & inr32;
            takef5 = !__any_sync(0xFFFFFFFFu, (F5 & nz) != 0u);
            F5 &= T32;
        }
        if (n_w) last_i = i;
        if (take2 || takef || takef5) {
            if (take2)
                lane_slots_2b<kDelta, kSwz, 8>(wp3, w, T32 & inr32, st_base + 4u * (a + wexcl), carry);
            else if (!kDelta && takef5)
                lane_slots_fast<kDelta, kSwz, true>(wp3, w, T32, st_base + 4u * (a + wexcl), carry, F5);
            else
                lane_slots_fast<kDelta, kSwz>(wp3, w, T32, st_base + 4u * (a + wexcl), carry);
            // the slice holds integer limit-1: record its end (stores past limit are
            // dropped by the copy-out)
            if (run < limit && run + n_w >= limit)
                slice_count_end(R, K, q0, T32 & inr32, static_cast<uint32_t>(limit - 1 - run), wexcl, n_own);
        } else
            carry = ll_slice_gen<kDelta, kSwz>(R, q0, x0, x1, wp2, wp3, T32, inr32, n_w, wexcl, run, limit, K,
                                               st_base + 4u * (a + wexcl), st_base + kSparseWin + 72u * lane, carry);
        if (n_w == 0) continue;
        __syncwarp();
        stage_out<kSwz>(st_base, a, n_w, run, limit, out, lane);
        run += n_w;
        __syncwarp();  // the staging buffer is rewritten by the next slice
    }
    // the end of the range's last integer: in slice last_i
    long long last_end = -1;
    if (last_i >= 0 && !K.hdr) {  // (a stream decode finds the stream's last integer in its completion)
        const long long q0 = qs + static_cast<long long>(kLLSlice) * last_i + 32 * lane;
        const uint4 x0 = r_load16(R, q0), x1 = r_load16(R, q0 + 16);
        const uint32_t e0 = hibits16(~x0.x, ~x0.y, ~x0.z, ~x0.w) & r_inr16(R, q0);
        const uint32_t e1 = hibits16(~x1.x, ~x1.y, ~x1.z, ~x1.w) & r_inr16(R, q0 + 16);
        if (e1) last_end = q0 + 16 + (31 - __clz(e1)) + 1 - R.lo;
        else if (e0) last_end = q0 + (31 - __clz(e0)) + 1 - R.lo;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const long long le = __shfl_xor_sync(0xFFFFFFFFu, last_end, o);
            last_end = le > last_end ? le : last_end;
        }
    }
    ro.last_end = last_end;
    ro.n = run - base;
    ro.carry = carry;
}

// 16-byte-lane range decode (delta); ring: the warp's input ring (2 x 512 bytes used).  Slices
// are indexed from qs; interior slices (inside [R.lo, R.hi)) arrive by
// cp.async one slice ahead into ring half (i & 1), the others are read with
// range masks.
template <bool kDelta, bool kSwz>
__device__ __forceinline__ void decode_range_ll16(const ByteRange& R, long long qs, long long qe,
                                                unsigned long long base, uint32_t carry, unsigned long long limit,
                                                uint32_t* out, uint32_t* stage, uint32_t ring, int lane,
                                                const RangeSink& K, RangeOut& ro) {
    const uint32_t out_w = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(out) >> 2);
    const uint32_t st_base = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
    const int ns = static_cast<int>((qe - qs + kSegSlice - 1) / kSegSlice);
    int i_lo, i_hi;  // interior slices: i_lo <= i < i_hi
    {
        const long long d = R.lo - qs, e = R.hi - qs;
        const long long lo = d <= 0 ? 0 : (d + kSegSlice - 1) / kSegSlice;
        const long long hi = e <= 0 ? 0 : e / kSegSlice;
        i_lo = static_cast<int>(lo < ns ? lo : ns);
        i_hi = static_cast<int>(hi < ns ? hi : ns);
    }
    const uint8_t* const pin = R.ab + qs + 16 * lane;  // this lane's bytes of slice 0
    const uint32_t rbase = ring + 16u * lane;
    // integers that may still be stored before `limit` (clamped): a slice with fewer takes the fast path
    uint32_t left;
    {
        const unsigned long long r = limit > base ? limit - base : 0ull;
        left = r > 0x7FFFFFFFull ? 0x7FFFFFFFu : static_cast<uint32_t>(r);
    }
    unsigned long long run = base;  // output index of the group's first integer
    int last_i = -1;                // the last slice holding an integer (warp-uniform)
    uint32_t pw3 = 0;               // lane 0: the 4 bytes before the slice
    if (lane == 0) pw3 = r_inside(R, qs - 4, 4) ? __ldg(reinterpret_cast<const uint32_t*>(R.ab + qs - 4))
                                                : r_word(R, qs - 4);
    if (i_lo == 0 && i_hi > 0) {
        cp_async16(rbase, pin);
        cp_async_commit();
    }
    for (int g = 0; g < ns; g += kLaneGroup) {
        const uint32_t a = (out_w + static_cast<uint32_t>(run)) & 3u;  // staging offset of the group
        uint32_t n_g = 0;
#pragma unroll 1
        for (int i = g; i < g + kLaneGroup && i < ns; ++i) {
            const bool inter = i >= i_lo && i < i_hi;  // warp-uniform
            const bool pfn = i + 1 >= i_lo && i + 1 < i_hi;
            if (pfn) {
                cp_async16(rbase + 512u * ((i + 1) & 1), pin + kSegSlice * (i + 1));
                cp_async_commit();
            }
            uint4 x;
            if (inter) {
                if (pfn) cp_async_wait<1>();
                else cp_async_wait<0>();
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w)
                             : "r"(rbase + 512u * (i & 1))
                             : "memory");
            } else {
                x = r_load16(R, qs + static_cast<long long>(kSegSlice) * i + 16 * lane);
            }
            const uint32_t w0 = x.x, w1 = x.y, w2 = x.z, w3 = x.w;
            uint32_t wp3 = __shfl_up_sync(0xFFFFFFFFu, w3, 1);
            const uint32_t l3 = __shfl_sync(0xFFFFFFFFu, w3, 31);
            if (lane == 0) wp3 = pw3;
            pw3 = l3;
            const uint32_t T16 = hibits16(~w0, ~w1, ~w2, ~w3);
            const uint32_t inr16 =
                inter ? 0xFFFFu : r_inr16(R, qs + static_cast<long long>(kSegSlice) * i + 16 * lane);
            const uint32_t n_own = __popc(T16 & inr16);
            uint32_t incl = n_own;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= o) incl += y;
            }
            const uint32_t n_w = __shfl_sync(0xFFFFFFFFu, incl, 31);
            const uint32_t wexcl = incl - n_own;
            // a tail slice (bytes past the range end only, read as 0x80: never
            // terminators) may take the 2-byte path too; its vote counts
            // continuation bytes inside the range only
            const bool tail = !inter && qs + static_cast<long long>(kSegSlice) * i >= R.lo;
            const uint32_t C20 =
                ~(hibits4(~wp3) | (T16 << 4)) &
                (inter ? 0xFFFFFu
                       : (inr16 << 4) | halo_in_range(R, qs + static_cast<long long>(kSegSlice) * i + 16 * lane));
            const uint32_t pair = C20 & (C20 >> 1);  // bit j: positions j-4, j-3 both continue
            const uint32_t run2 = pair & 0xFFFFCu;     // a 3+-byte integer ends in 0..15
            const uint32_t run4 = pair & (pair >> 2);  // a 5+-byte integer ends in 0..15
            const unsigned vote = (__any_sync(0xFFFFFFFFu, run2 != 0) ? 1u : 0u) | (__any_sync(0xFFFFFFFFu, run4 != 0) ? 2u : 0u);
            const bool take2 = (inter || tail || MVB_HEAD2) && vote == 0;  // (head slices: see decode_range_ll)
            const bool takef = !take2 && inter && !(vote & 2u);
            if (n_w) last_i = i;
            if (take2 || takef) {
                if (take2) {
                    const uint32_t wv[4] = {w0, w1, w2, w3};
                    lane_slots_2b<kDelta, kSwz, 4>(wp3, wv, T16 & inr16, st_base + 4u * (a + n_g + wexcl), carry);
                } else {
                    lane_slots_fast16<kDelta, kSwz>(wp3, w0, w1, w2, w3, T16, st_base + 4u * (a + n_g + wexcl), carry);
                }
                // the slice holds integer limit-1: record its end (stores past limit are
                // dropped by the copy-out)
                if (left > 0 && n_w >= left)
                    slice_count_end(R, K, qs + static_cast<long long>(kSegSlice) * i + 16 * lane, T16 & inr16,
                                    left - 1, wexcl, n_own);
            } else
                carry = ll_slice_gen16<kDelta, kSwz>(R, qs + static_cast<long long>(kSegSlice) * i + 16 * lane, w0,
                                                     w1, w2, w3, wp3, T16, inr16, n_own, n_w, wexcl, run + n_g, limit,
                                                     K, st_base + 4u * (a + n_g + wexcl), carry);
            n_g += n_w;
            left = left > n_w ? left - n_w : 0u;
        }
        if (n_g == 0) continue;
        __syncwarp();
        stage_out<kSwz>(st_base, a, n_g, run, limit, out, lane);
        run += n_g;
        __syncwarp();  // the staging buffer is rewritten by the next group
    }
    // the end of the range's last integer: in slice last_i
    long long last_end = -1;
    if (last_i >= 0 && !K.hdr) {  // (a stream decode finds the stream's last integer in its completion)
        const long long q0 = qs + static_cast<long long>(kSegSlice) * last_i + 16 * lane;
        const uint4 x = r_load16(R, q0);
        const uint32_t e16 = hibits16(~x.x, ~x.y, ~x.z, ~x.w) & r_inr16(R, q0);
        if (e16) last_end = q0 + (31 - __clz(e16)) + 1 - R.lo;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const long long le = __shfl_xor_sync(0xFFFFFFFFu, last_end, o);
            last_end = le > last_end ? le : last_end;
        }
    }
    ro.last_end = last_end;
    ro.n = run - base;
    ro.carry = carry;
}

// The lane-local range decode: 32-byte lanes (half the per-slice fixed work
// per byte of 16-byte lanes); batched delta lists keep 16-byte lanes.
template <bool kDelta, bool kSwz>
__device__ __forceinline__ void decode_range_llw(const ByteRange& R, long long qs, long long qe,
                                                 unsigned long long base, uint32_t carry, unsigned long long limit,
                                                 uint32_t* out, uint32_t* stage, uint32_t ring, int lane,
                                                 const RangeSink& K, RangeOut& ro) {
    // (batched lists -- K.hdr null -- keep 16-byte lanes for delta: most lists are
    // short, and 1 KiB slices would mostly be padding)
    if (kDelta && (!MVB_DELTA32 || !K.hdr))
        decode_range_ll16<kDelta, kSwz>(R, qs, qe, base, carry, limit, out, stage, ring, lane, K, ro);
    else
        decode_range_ll<kDelta, kSwz>(R, qs, qe, base, carry, limit, out, stage, ring, lane, K, ro);
}

// Completion of a kernel-B launch (all threads of every CTA call it): the
// last CTA to arrive sums the launch's group totals and re-zeroes the
// launch's group / supergroup accumulators; a non-final launch of a pipelined
// decode publishes the totals before s_hi, the final one produces the
// DecodeResult and resets the header.  find_last_end: the end of the stream's
// last integer (needed only for a truncated stream) is found here -- the last
// segment with an integer, then its last terminator byte -- instead of being
// tracked by every range decode.
template <int kNW>
__device__ __forceinline__ void seg_complete(const SegParams& S, bool find_last_end) {
    __shared__ bool s_last;
    __shared__ unsigned long long s_tot[kNW], s_sum[kNW];
    __shared__ long long s_seg;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&S.hdr->done, 1ull) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // integer count and value sum of the groups before s_hi; then zero this
    // launch's group accumulators for the next launch
    const long long g_lo = S.s_lo >> 5, g_hi = (S.s_hi + 31) >> 5;
    unsigned long long tot = 0, tsum = 0;
    for (long long k = g_lo + threadIdx.x; k < g_hi; k += blockDim.x) {
        tot += S.gcnt[k];
        tsum += S.gsum[k];
        S.gcnt[k] = 0;
        S.gsum[k] = 0;
    }
    // supergroups the launch touched (one straddling two chunks of a pipelined
    // decode is never read whole; both launches zero it)
    for (long long k = (g_lo >> 5) + threadIdx.x; k < ((g_hi + 31) >> 5); k += blockDim.x) {
        S.ucnt[k] = 0;
        S.usum[k] = 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        tot += __shfl_xor_sync(0xFFFFFFFFu, tot, o);
        tsum += __shfl_xor_sync(0xFFFFFFFFu, tsum, o);
    }
    if (lane == 0) {
        s_tot[wid] = tot;
        s_sum[wid] = tsum;
    }
    if (threadIdx.x == 0) s_seg = -1;
    __syncthreads();
    unsigned long long total = S.base_in ? S.base_in[0] : 0ull, sum = S.base_in ? S.base_in[1] : 0ull;
    for (int k = 0; k < kNW; ++k) {
        total += s_tot[k];
        sum += s_sum[k];
    }
    if (!S.final_launch) {  // a chunk of a pipelined decode: publish, keep the header
        if (threadIdx.x == 0) {
            S.base_out[0] = total;
            S.base_out[1] = sum;
            if (S.chunk_total) {
                *S.chunk_total = total;
                __threadfence_system();
            }
            S.hdr->done = 0;
            S.hdr->ticket = 0;
        }
        return;
    }
    WsHeader* h = S.hdr;
    const unsigned long long err_inv = *reinterpret_cast<volatile unsigned long long*>(&h->err_idx_inv);
    const bool truncated = !(err_inv != 0ull && ~err_inv < S.count) && total < S.count;  // (CTA-uniform)
    long long last_end_found = 0;
    if (find_last_end && truncated) {
        for (long long hi = S.n_seg - 1; hi >= 0; hi -= blockDim.x) {
            const long long k = hi - static_cast<long long>(threadIdx.x);
            if (k >= 0 && S.scnt[k] > 0) atomicMax(&s_seg, k);
            __syncthreads();
            if (s_seg >= 0) break;
        }
        if (s_seg >= 0) {
            // its last terminator byte: blocks of 16 bytes per thread, from the
            // segment's end (clipped to the stream) backwards until one holds it
            __shared__ long long s_le;
            const long long p_lo = s_seg * S.seg_bytes - S.mis > 0 ? s_seg * S.seg_bytes - S.mis : 0;
            long long p_hi = (s_seg + 1) * S.seg_bytes - S.mis;
            if (p_hi > S.len) p_hi = S.len;
            for (long long top = p_hi; top > p_lo; top -= 16ll * blockDim.x) {
                if (threadIdx.x == 0) s_le = -1;
                __syncthreads();
                const long long b = top - 16ll * (threadIdx.x + 1);
                long long le = -1;
                for (int j = 15; j >= 0 && le < 0; --j) {
                    const long long p = b + j;
                    if (p >= p_lo && p < p_hi && S.in[p] < 0x80u) le = p + 1;
                }
                if (le >= 0) atomicMax(&s_le, le);
                __syncthreads();
                if (s_le >= 0) break;
            }
            if (threadIdx.x == 0) last_end_found = s_le > 0 ? s_le : 0;
        }
    }
    if (!S.base_in) {  // whole-stream launch: zero the segment totals (a pipelined decode's host memsets them)
        __syncthreads();
        for (long long k = S.s_lo + threadIdx.x; k < S.s_hi; k += blockDim.x) {
            S.scnt[k] = 0;
            S.ssum[k] = 0;
        }
    }
    if (threadIdx.x == 0) {
        const unsigned long long errpos_inv = *reinterpret_cast<volatile unsigned long long*>(&h->err_pos_inv);
        const unsigned long long last_end =
            find_last_end ? static_cast<unsigned long long>(last_end_found)
                          : *reinterpret_cast<volatile unsigned long long*>(&h->last_end);
        const unsigned long long count_end = *reinterpret_cast<volatile unsigned long long*>(&h->count_end);
        mvb_result r;
        r.reserved = 0;
        if (err_inv != 0ull && ~err_inv < S.count) {
            r.status = MVB_MALFORMED;
            r.values_written = ~err_inv;
            r.bytes_consumed = ~errpos_inv;
        } else if (total >= S.count) {
            r.status = MVB_OK;
            r.values_written = S.count;
            r.bytes_consumed = count_end;
        } else {
            r.status = MVB_TRUNCATED;
            r.values_written = total;
            r.bytes_consumed = last_end;
        }
        h->result = r;
        if (S.res_dev) *S.res_dev = r;
        h->done = 0;
        h->ticket = 0;
        h->err_idx_inv = 0;
        h->err_pos_inv = 0;
        h->last_end = 0;
        h->count_end = 0;
        h->epoch = h->epoch + 1;
    }
    __threadfence();
}

// Integer count and digit-weight sum of the stream before segment s (all
// lanes get them): the launch's base, whole supergroups and the partial
// groups at both ends of [g_lo, g), the segments before s in its group --
// independent loads, one memory latency.
template <bool kDelta>
__device__ __forceinline__ void seg_prefix(const SegParams& S, long long s, int lane, unsigned long long& base,
                                           unsigned long long& csum) {
    base = 0;
    csum = 0;
    const long long g = s >> 5, g_lo = S.s_lo >> 5;
    if (lane == 0 && S.base_in) {
        base = S.base_in[0];
        csum = S.base_in[1];
    }
    const long long ua = (g_lo + 31) >> 5, ub = g >> 5;  // whole supergroups [ua, ub)
    if (ua < ub) {
        const long long h = g_lo + lane, t = (ub << 5) + lane;
        if (h < (ua << 5)) {
            base += S.gcnt[h];
            if (kDelta) csum += S.gsum[h];
        }
        if (t < g) {
            base += S.gcnt[t];
            if (kDelta) csum += S.gsum[t];
        }
        for (long long k = ua + lane; k < ub; k += 32) {
            base += S.ucnt[k];
            if (kDelta) csum += S.usum[k];
        }
    } else {
        for (long long k = g_lo + lane; k < g; k += 32) {
            base += S.gcnt[k];
            if (kDelta) csum += S.gsum[k];
        }
    }
    if (lane < (s & 31)) {
        base += S.scnt[(g << 5) + lane];
        if (kDelta) csum += S.ssum[(g << 5) + lane];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        base += __shfl_xor_sync(0xFFFFFFFFu, base, o);
        if (kDelta) csum += __shfl_xor_sync(0xFFFFFFFFu, csum, o);
    }
}

template <bool kDelta>
__global__ void __launch_bounds__(kSegThreads, kDelta ? kLLBlocksD : kLLBlocks) vbyte_seg_decode(SegParams S) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    char* const vbase = reinterpret_cast<char*>(smem) + wid * kLaneWarpBytes;
    const uint32_t ring = static_cast<uint32_t>(__cvta_generic_to_shared(vbase + 4 * kLaneStage));
    const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    const ByteRange R = {S.in - S.mis, S.mis, S.mis + S.len, S.mis, S.mis + S.len};
    // one contiguous run of segments per warp (the output index and carry after
    // segment s are those of s + 1, so only the run's first segment needs the
    // prefix)
    const long long ns = S.s_hi - S.s_lo;
    const long long s0 = S.s_lo + gw * ns / nw, s_step = ns;
    const long long s0_end = S.s_lo + (gw + 1) * ns / nw;  // balanced runs: sizes differ by at most one
    // kernel A's totals are complete and visible after this (a no-op unless
    // launched as a programmatic dependent)
    asm volatile("griddepcontrol.wait;" ::: "memory");
#if MVB_A_PDL
    // the next decode's kernel A may start its loads as this grid's CTAs retire
    // (it waits for this grid before its first write)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif

    for (long long s = s0; s < s0_end; s += s_step) {
        const long long s_end = s0_end;
        // ---- output index and carry of the segment ----
        unsigned long long base, csum;
        seg_prefix<kDelta>(S, s, lane, base, csum);
        if (base >= S.count) continue;  // nothing of this segment is stored (warp-uniform)
        // segment sums are digit-weight sums of the segments' bytes: the bytes before
        // this segment that belong to the integer straddling its start (the partial
        // value of the <= 4 bytes after the last terminator before it) are not yet
        // an integer of the prefix
        uint32_t straddle = 0;
        if (kDelta) {
            const uint32_t wb = r_word(R, s * S.seg_bytes - 4);
            straddle = shr_clamp(pack28(wb), 7 * (32 - __clz(static_cast<int>(hibits4(~wb)))));
        }
        const uint32_t carry =
            kDelta ? static_cast<uint32_t>(csum) - straddle + (S.prev_dev ? S.prev + *S.prev_dev : S.prev) : 0u;
        RangeOut ro;
        const RangeSink K = {S.hdr, nullptr, nullptr, nullptr};
        {
            // integers in the run (segments s .. s_end - 1, at most 32): its density
            unsigned long long rc = (s + lane < s_end) ? S.scnt[s + lane] : 0u;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) rc += __shfl_xor_sync(0xFFFFFFFFu, rc, o);
            // the last segment ends with the stream (no slices of padding: they hold no
            // integer and would all take the masked general path)
            const long long q_stream_end = (R.hi + 15) & ~15ll;
            const long long qe = s_end * S.seg_bytes < q_stream_end ? s_end * S.seg_bytes : q_stream_end;
            if (range_dense(rc, qe - s * S.seg_bytes))
                decode_range_llw<kDelta, true>(R, s * S.seg_bytes, qe, base, carry, S.count, S.out,
                                              reinterpret_cast<uint32_t*>(vbase), ring, lane, K, ro);
            else
                decode_range_llw<kDelta, false>(R, s * S.seg_bytes, qe, base, carry, S.count, S.out,
                                               reinterpret_cast<uint32_t*>(vbase), ring, lane, K, ro);
        }
    }

    // ---- completion; the last CTA produces the DecodeResult ----
    seg_complete<kSegWarps>(S, true);
}

// ------------------------------------------------------------------ batched lists

// Independent lists (BASELINE config 3, SURVEY.md §8e "c3: independent
// units"): list l is the byte span in[byte_off[l] .. byte_off[l+1]) holding
// int_off[l+1] - int_off[l] integers, decoded -- delta from prev[l] (0 if no
// prev array) -- into out[int_off[l] ...], exactly as the reference's
// per-list decode_delta_stream call (tools/bench/runner.cpp:28-61) would.
// One warp per list, lists handed out by a ticket counter (in `order` if
// given, e.g. longest first); no cross-list dependency at all.
struct ListParams {
    const uint8_t* ab;  // 16-byte-aligned base: in = ab + mis0
    long long mis0;
    long long in_len;
    const unsigned long long* byte_off;  // n_lists + 1
    const unsigned long long* int_off;   // n_lists + 1
    const uint32_t* prev;                // n_lists or null
    const unsigned* order;               // n_lists or null
    long long n_lists;
    uint32_t* out;
    mvb_result* results;  // n_lists or null
    WsHeader* hdr;
};

template <bool kDelta>
__global__ void __launch_bounds__(kSegThreads, kDelta ? kLLBlocksD : kLLBlocks) vbyte_lists_decode(ListParams L) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ bool s_last;
    __shared__ unsigned long long s_err_idx[kSegWarps];
    __shared__ long long s_err_pos[kSegWarps], s_count_end[kSegWarps];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    char* const vbase = reinterpret_cast<char*>(smem) + wid * kLaneWarpBytes;
    const uint32_t ring = static_cast<uint32_t>(__cvta_generic_to_shared(vbase + 4 * kLaneStage));
    while (true) {
        long long k = 0;
        if (lane == 0) k = static_cast<long long>(atomicAdd(&L.hdr->ticket, 1ull));
        k = __shfl_sync(0xFFFFFFFFu, k, 0);
        if (k >= L.n_lists) break;
        const long long l = L.order ? static_cast<long long>(L.order[k]) : k;
        long long b0 = static_cast<long long>(L.byte_off[l]), b1 = static_cast<long long>(L.byte_off[l + 1]);
        if (b1 > L.in_len) b1 = L.in_len;  // never read past in + in_len
        if (b0 > b1) b0 = b1;
        const unsigned long long base = L.int_off[l];
        const unsigned long long cnt = L.int_off[l + 1] > base ? L.int_off[l + 1] - base : 0ull;
        mvb_result r;
        r.reserved = 0;
        if (cnt == 0) {  // decode_test.cpp:204-206: an empty request is OK
            r.status = MVB_OK;
            r.values_written = 0;
            r.bytes_consumed = 0;
        } else {
            const ByteRange R = {L.ab, L.mis0 + b0, L.mis0 + b1, L.mis0, L.mis0 + L.in_len};
            if (lane == 0) {
                s_err_idx[wid] = ~0ull;
                s_count_end[wid] = -1;
            }
            __syncwarp();
            RangeOut ro;
            const RangeSink K = {nullptr, &s_err_idx[wid], &s_err_pos[wid], &s_count_end[wid]};
            const uint32_t carry = kDelta && L.prev ? L.prev[l] : 0u;
            if (range_dense(cnt, R.hi - R.lo))
                    decode_range_llw<kDelta, true>(R, R.lo & ~15ll, R.hi, base, carry, base + cnt, L.out,
                                                  reinterpret_cast<uint32_t*>(vbase), ring, lane, K, ro);
                else
                    decode_range_llw<kDelta, false>(R, R.lo & ~15ll, R.hi, base, carry, base + cnt, L.out,
                                                   reinterpret_cast<uint32_t*>(vbase), ring, lane, K, ro);

            __syncwarp();
            const unsigned long long ei = s_err_idx[wid];
            if (ei != ~0ull && ei < base + cnt) {
                r.status = MVB_MALFORMED;
                r.values_written = ei - base;
                r.bytes_consumed = static_cast<unsigned long long>(s_err_pos[wid]);
            } else if (ro.n >= cnt) {
                r.status = MVB_OK;
                r.values_written = cnt;
                r.bytes_consumed = static_cast<unsigned long long>(s_count_end[wid]);
            } else {
                r.status = MVB_TRUNCATED;
                r.values_written = ro.n;
                r.bytes_consumed = ro.last_end >= 0 ? static_cast<unsigned long long>(ro.last_end) : 0ull;
            }
        }
        if (lane == 0 && L.results) L.results[l] = r;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&L.hdr->done, 1ull) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        L.hdr->ticket = 0;
        L.hdr->done = 0;
        __threadfence();
    }
}

}  // namespace mvbk
