// decode_fused.cuh -- the default strict-mode stream decoder: one persistent
// kernel that reads the compressed stream from HBM exactly once.
//
// The stream (16-byte-aligned coordinates q = p + mis) is cut into units of
// kUnit bytes.  Each warp owns a shared-memory buffer for one unit and takes
// units u = 0, 1, 2, ... from a ticket counter:
//
//   load      one TMA bulk copy (cp.async.bulk + mbarrier) of the unit and the
//             16 bytes before it into the warp's buffer (units at the stream's
//             edges: masked loads);
//   A(u)      the unit's terminator count and digit-weight sum, from shared
//             memory (SegParams convention: the sums before a unit are the
//             value sum of the integers before it plus the partial value of
//             the integer straddling its start), published to a 32-ary tree of
//             partial sums (level 0 = units, level l = blocks of 32^l units);
//   prefix    the unit's output index and delta carry: the sums of at most 31
//             published entries per level (one memory latency; the units
//             before u took their tickets earlier, so their totals are out or
//             about to be);
//   B(u)      the lane-local decode (decode_range_ll's per-slice algorithm) of
//             the unit's 1 KiB slices straight from the buffer, values staged
//             per slice and copied out as 16-byte-aligned quads.
//
// Nothing but the tree's 16-byte entries and the output leaves the SM, and the
// input crosses HBM once (the two-kernel decoder, decode_seg.cuh, read it
// twice: its kernel B found the bytes in L2 only for streams up to ~100 MB).
//
// Tree entries are two 64-bit words, each carrying the launch's epoch as a
// 24-bit tag next to its value (count << 24 | tag, sum << 32 | tag): a word
// is written and read in one access, so a reader that sees this launch's tag
// in both has the values -- no fences, and nothing is zeroed between
// launches.  An entry is aggregated by the last of its children to arrive
// (per-entry arrival counters only grow: every launch adds exactly the
// entry's child count).  The last CTA to finish produces the DecodeResult
// (fused_complete).  All CTAs must be co-resident (the grid is sized from the
// occupancy calculator): a unit waits for the totals of every unit before it.
//
// Replaces the reference's stream loop (stream_loop.hpp:31-129) for
// DecodeMode::strict with the semantics of decode_scalar / decode_delta_scalar
// (vbyte.cpp:47-74, internal.hpp:22-37).
#pragma once

#include "decode_seg.cuh"

namespace mvbk {

#ifndef MVB_F_UNIT
#define MVB_F_UNIT 4096  // bytes per unit (a multiple of 1 KiB)
#endif
#ifndef MVB_BULK_OUT
#define MVB_BULK_OUT 1  // copy-out of plain-layout staging by TMA bulk copies (0: ld.shared / st.global quads)
#endif
#ifndef MVB_F_PF
#define MVB_F_PF 8  // L2 prefetch distance of the unit loads, in eighths of a round of tickets (0: none)
#endif
#ifndef MVB_F_PF0
#define MVB_F_PF0 1  // rounds of units prefetched into L2 before the wait for the previous grid
#endif
#ifndef MVB_F_STATIC0
#define MVB_F_STATIC0 8  // streams of fewer than this many units per warp: the first round of units without tickets (0: never)
#endif
#ifndef MVB_OUT_PRED
#define MVB_OUT_PRED 1  // the d3 copy-out as predicated instructions instead of branches (c4 987 -> 932 us)
#endif
#ifndef MVB_F_SLEEP
#define MVB_F_SLEEP 32  // ns between two looks at a tree entry not yet published
#endif
#ifndef MVB_F_LATE
#define MVB_F_LATE 0  // 1: a unit's prefix entries are checked (and waited for) after the next unit's publication
#endif
#ifndef MVB_F_BLOCKS
#define MVB_F_BLOCKS 4  // resident CTAs per SM (shared memory: one unit buffer + staging per warp)
#endif
constexpr int kFBlocks = MVB_F_BLOCKS;
constexpr int kUnit = MVB_F_UNIT;
constexpr int kUnitBuf = (16 + kUnit + 127) / 128 * 128;      // 16 halo bytes + the unit
constexpr int kFStage = 1152;                                 // staging words: a slice of <= 1120 integers + alignment
static_assert(kFStage >= kLaneStage, "staging serves decode_unit_ll too");
constexpr int kFWarpBytes = 2 * kUnitBuf + 4 * kFStage;       // two unit buffers + the slice staging
constexpr int kFSmem = kSegWarps * kFWarpBytes + 16 * kSegWarps;  // + two mbarriers per warp
constexpr int kFLevels = 6;                                   // tree levels: up to 32^6 units
static_assert(kUnit % 1024 == 0 && kFWarpBytes % 128 == 0, "unit geometry");

// One tree entry: (count << 24 | tag), (sum << 32 | tag); tag = epoch mod 2^24.
struct alignas(16) FEntry {
    unsigned long long c;
    unsigned long long s;
};

struct FusedParams {
    SegParams S;                 // in, mis, len, count, out, prev, prev_dev, seg_bytes (= kUnit), n_seg, hdr, res_dev
    int swz;                     // staging swizzle: 0 never, 1 always, 2 dense units (debug switch)
    int narrow;                  // every count fits 32 bits (stream < 4 GiB): warp sums by redux
    int mode;                    // 0 totals and decode, 1 totals only (-> rec), 2 decode only (totals of a mode-1 launch)
    unsigned long long* rec;     // mode 1: the stream's [integer count, value sum]
    int levels;                  // tree levels in use (32^levels >= n_seg)
    long long n_at[kFLevels];    // entries per level (n_at[0] = n_seg)
    FEntry* tree[kFLevels];      // level arrays
    unsigned* arrive[kFLevels];  // per entry of levels >= 1: arrivals over all launches
};

// Digit-weight sum and continuation count of one word w (p = the word
// before it), for streams whose integers have at most 3 bytes: a byte after
// k continuation bytes weighs 128^k; classes 0/1 (weights 1 / 128) in one
// dp4a, class 2 (2^14) in a second.  hi3 collects the bytes after three
// continuation bytes (the caller then redoes the iteration exactly).
__device__ __forceinline__ void ftot_word(uint32_t w, uint32_t p, uint32_t& cc, uint32_t& sA, uint32_t& sB,
                                          uint32_t& hi3) {
    const uint32_t ck = w & 0x80808080u, cp = p & 0x80808080u;
    cc = __dp4a(ck, 0x01010101u, cc);                        // 128 per continuation byte
    const uint32_t c1 = __funnelshift_l(cp, ck, 1);          // bit 0 of byte j: byte j-1 continues
    const uint32_t c2 = c1 & __funnelshift_l(cp, ck, 9);     // ... and byte j-2
    hi3 |= c2 & __funnelshift_l(cp, ck, 17);                 // ... and byte j-3
    const uint32_t wa = c1 * 127u + 0x01010101u - c2 * 128u;  // 1, 128, or 0 (class 2)
    const uint32_t w7 = w & 0x7F7F7F7Fu;
    sA = __dp4a(w7, wa, sA);
    sB = __dp4a(w7, c2, sB);
}

// The exact digit-weight sum of word w given the 8 bytes before it (p1 =
// the word before, p2 = the one before that): weights 128^k for k = 0..4
// continuation bytes before, 0 for five or more (2^35 = 0 mod 2^32).
__device__ __forceinline__ uint32_t ftot_word_exact(uint32_t w, uint32_t p1, uint32_t p2) {
    const uint32_t ck = w & 0x80808080u, c1p = p1 & 0x80808080u, c2p = p2 & 0x80808080u;
    const uint32_t c1 = __funnelshift_l(c1p, ck, 1);
    const uint32_t c2 = c1 & __funnelshift_l(c1p, ck, 9);
    const uint32_t c3 = c2 & __funnelshift_l(c1p, ck, 17);
    const uint32_t c4 = c3 & __funnelshift_l(c1p, ck, 25);
    const uint32_t c5 = c4 & __funnelshift_l(c2p, c1p, 1);
    const uint32_t w7 = w & 0x7F7F7F7Fu;
    const uint32_t wa = c1 * 127u + 0x01010101u - c2 * 128u;  // classes 0, 1
    const uint32_t wb = c2 + c3 * 127u - c4 * 128u;            // classes 2, 3 (x 2^14)
    const uint32_t wc = c4 - c5;                                // class 4 (x 2^28)
    return __dp4a(w7, wa, 0u) + (__dp4a(w7, wb, 0u) << 14) + (__dp4a(w7, wc, 0u) << 28);
}

// 16 bytes through the non-coherent path with an L2 evict-last policy (the
// bytes are read again from L2 by the segment's decode, D units later)
__device__ __forceinline__ uint4 ldg_keep16(const void* p, unsigned long long pol) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}

// Terminator count (inside the stream) and, for delta, digit-weight sum of
// the segment bytes [q0, q1) (1 KiB iterations; lane l: bytes 32l .. 32l+31
// of each).  Identical in every lane on return.
// flags_out bit 0 (delta): some byte follows three or more continuation bytes
// (an integer of 4+ bytes, or a malformed run).
template <bool kDelta>
__device__ __forceinline__ void fused_totals(const SegParams& S, long long q0, long long q1, int lane,
                                             unsigned& cnt_out, uint32_t& sum_out, uint32_t ubuf = 0u,
                                             uint32_t* flags_out = nullptr) {
    const uint8_t* const ab = S.in - S.mis;
    const long long qlo = S.mis, qhi = S.mis + S.len;
    // ubuf: shared-memory address of byte q0 (the whole range and the 16 bytes
    // before it are there, inside the stream), or 0: read global memory
    uint32_t h1 = 0, h2 = 0;  // lane 0: the 8 bytes before the iteration (word -1, word -2)
    if (lane == 0) {
        if (ubuf) {
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(h2), "=r"(h1) : "r"(ubuf - 8u) : "memory");
        } else {
            h1 = seg_word(S, q0 - 4);
            h2 = seg_word(S, q0 - 8);
        }
    }
    unsigned tc = 0;      // terminators counted directly (edge iterations) + 32 per interior iteration
    uint32_t cc = 0;      // 128 x continuation bytes of interior iterations
    uint32_t sA = 0, sB = 0, sX = 0, flags = 0;
    long long q = q0;
    const unsigned long long pol = l2_evict_last();
    uint4 x0, x1;
    bool in0 = q >= qlo && q + 1024 <= qhi;
    if (q < q1) {
        const long long ql = q + 32 * lane;
        if (ubuf) {
            x0 = lds128(ubuf + static_cast<uint32_t>(ql - q0));
            x1 = lds128(ubuf + static_cast<uint32_t>(ql - q0) + 16u);
        } else if (in0) {
            x0 = ldg_keep16(ab + ql, pol);
            x1 = ldg_keep16(ab + ql + 16, pol);
        } else {
            x0 = seg_load16(S, ql);
            x1 = seg_load16(S, ql + 16);
        }
    }
    for (; q < q1; q += 1024) {
        const uint32_t w[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        const bool inside = in0;
        // prefetch the next iteration
        const long long qn = q + 1024;
        in0 = qn >= qlo && qn + 1024 <= qhi;
        if (qn < q1) {
            const long long ql = qn + 32 * lane;
            if (ubuf) {
                x0 = lds128(ubuf + static_cast<uint32_t>(ql - q0));
                x1 = lds128(ubuf + static_cast<uint32_t>(ql - q0) + 16u);
            } else if (in0) {
                x0 = ldg_keep16(ab + ql, pol);
                x1 = ldg_keep16(ab + ql + 16, pol);
            } else {
                x0 = seg_load16(S, ql);
                x1 = seg_load16(S, ql + 16);
            }
        }
        uint32_t p1 = __shfl_up_sync(0xFFFFFFFFu, w[7], 1), p2 = __shfl_up_sync(0xFFFFFFFFu, w[6], 1);
        const uint32_t l1 = __shfl_sync(0xFFFFFFFFu, w[7], 31), l2 = __shfl_sync(0xFFFFFFFFu, w[6], 31);
        if (lane == 0) {
            p1 = h1;
            p2 = h2;
        }
        h1 = l1;
        h2 = l2;
        if (inside) {
            tc += 32;
        } else {
            const long long ql = q + 32 * lane;
            tc += __popc(hibits16(~w[0], ~w[1], ~w[2], ~w[3]) & seg_inr16(S, ql)) +
                  __popc(hibits16(~w[4], ~w[5], ~w[6], ~w[7]) & seg_inr16(S, ql + 16));
        }
        if (kDelta) {
            uint32_t hi3 = 0, a = 0, b = 0, ccx = 0;
            ftot_word(w[0], p1, ccx, a, b, hi3);
#pragma unroll
            for (int k = 1; k < 8; ++k) ftot_word(w[k], w[k - 1], ccx, a, b, hi3);
            if (__any_sync(0xFFFFFFFFu, hi3 != 0)) {  // an integer of 4+ bytes: the exact weights
                flags |= 1u;
                uint32_t s = ftot_word_exact(w[0], p1, p2) + ftot_word_exact(w[1], w[0], p1);
#pragma unroll
                for (int k = 2; k < 8; ++k) s += ftot_word_exact(w[k], w[k - 1], w[k - 2]);
                sX += s;
            } else {
                sA += a;
                sB += b;
            }
            if (inside) cc += ccx;
        } else if (inside) {
#pragma unroll
            for (int k = 0; k < 8; ++k) cc = __dp4a(w[k] & 0x80808080u, 0x01010101u, cc);
        }
    }
    if (flags_out) *flags_out = flags;
    unsigned cnt = tc - (cc >> 7);
    cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
    uint32_t sum = 0;
    if (kDelta) sum = __reduce_add_sync(0xFFFFFFFFu, sA + (sB << 14) + sX);
    cnt_out = cnt;
    sum_out = sum;
}

// ---- delta slices whose integers have at most 3 bytes (c2, c4: nearly every slice) ----
//
// Every byte b contributes d(b) * 128^k to the running sum, k = the number of
// continuation bytes right before it (0..2 here), so the delta output at
// terminator t is carry + (the sum of all contributions up to t): one dp2a
// per byte (two 16-bit weights x two digit bytes, plus an accumulator),
// with the previous output as the accumulator.  No integer value is ever
// assembled.  The carry of this path counts every byte before the slice
// (including the partial integer straddling into it); the other paths count
// complete integers only, so the carry is converted at entry and exit.

__device__ __forceinline__ uint32_t dp2a_lo(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("dp2a.lo.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t dp2a_hi(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("dp2a.hi.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
// The partial value of the bytes of word x after its last terminator (all
// four if it has none): the part of an integer that continues past x.
__device__ __forceinline__ uint32_t tail_value(uint32_t x) {
    return shr_clamp(pack28(x), 7 * (32 - __clz(static_cast<int>(hibits4(~x)))));
}

// One predicated staging store: if bit `bit` of T is set, stage[sp] = v, sp += 4.
template <bool kSwz>
__device__ __forceinline__ void slot_store(uint32_t& sp, uint32_t T, uint32_t bit, uint32_t v) {
    if (kSwz)
        asm volatile(
            "{\n\t.reg .pred p;\n\t.reg .b32 t, a;\n\t"
            "and.b32 t, %1, %2;\n\tsetp.ne.b32 p, t, 0;\n\t"
            "shr.b32 a, %0, 3;\n\tand.b32 a, a, 0x70;\n\txor.b32 a, a, %0;\n\t"
            "@p st.shared.u32 [a], %3;\n\t@p add.u32 %0, %0, 4;\n\t}"
            : "+r"(sp)
            : "r"(T), "r"(bit), "r"(v)
            : "memory");
    else
        asm volatile(
            "{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
            "and.b32 t, %1, %2;\n\tsetp.ne.b32 p, t, 0;\n\t"
            "@p st.shared.u32 [%0], %3;\n\t@p add.u32 %0, %0, 4;\n\t}"
            : "+r"(sp)
            : "r"(T), "r"(bit), "r"(v)
            : "memory");
}

// wp3: the 4 bytes before the lane; w: its 32 bytes; T: its in-range
// terminators (bit j = byte j); sp: staging address of its first output;
// carry (in/out, warp-uniform): the byte-convention carry before the slice.
// The word totals are independent dp2a pairs, so each word's outputs hang off
// its own base (short dependency chains instead of one chain of 16 dp2a).
template <bool kSwz>
__device__ __forceinline__ void lane_slots_d3(uint32_t wp3, const uint32_t (&w)[8], uint32_t T, uint32_t sp,
                                              uint32_t& carry) {
    uint32_t W01[8], W23[8], w7[8], tk[8];
    uint32_t prev = wp3;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t s8 = __funnelshift_l(prev, w[k], 8), s16 = __funnelshift_l(prev, w[k], 16);
        // byte j: 1 if byte j-1 continues, 0x81 if bytes j-1 and j-2 do
        const uint32_t x = ((s8 >> 7) & 0x01010101u) | (s8 & s16 & 0x80808080u);
        // 16-bit weights 1 + 127 x: 1, 128, 16384
        W01[k] = prmt_sign(x, 0u, 0x4140u) * 127u + 0x00010001u;
        W23[k] = prmt_sign(x, 0u, 0x4342u) * 127u + 0x00010001u;
        w7[k] = w[k] & 0x7F7F7F7Fu;
        tk[k] = dp2a_lo(W01[k], w7[k], dp2a_hi(W23[k], w7[k], 0u));
        prev = w[k];
    }
    uint32_t tot = tk[0];
#pragma unroll
    for (int k = 1; k < 8; ++k) tot += tk[k];
    uint32_t acc = lane_scan_offset<true>(tot, carry);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t o0 = dp2a_lo(W01[k] & 0xFFFFu, w7[k], acc);
        const uint32_t o1 = dp2a_lo(W01[k], w7[k], acc);
        const uint32_t o2 = dp2a_hi(W23[k] & 0xFFFFu, w7[k], o1);
        acc += tk[k];
        slot_store<kSwz>(sp, T, 1u << (4 * k), o0);
        slot_store<kSwz>(sp, T, 2u << (4 * k), o1);
        slot_store<kSwz>(sp, T, 4u << (4 * k), o2);
        slot_store<kSwz>(sp, T, 8u << (4 * k), acc);
    }
}

// One predicated staging store keyed on word w: if byte `bit` of w is a
// terminator (its high bit, given as the mask, clear), stage[sp] = v, sp += 4.
template <bool kSwz>
__device__ __forceinline__ void slot_store_w(uint32_t& sp, uint32_t w, uint32_t hibit, uint32_t v) {
    if (kSwz)
        asm volatile(
            "{\n\t.reg .pred p;\n\t.reg .b32 t, a;\n\t"
            "and.b32 t, %1, %2;\n\tsetp.eq.b32 p, t, 0;\n\t"
            "shr.b32 a, %0, 3;\n\tand.b32 a, a, 0x70;\n\txor.b32 a, a, %0;\n\t"
            "@p st.shared.u32 [a], %3;\n\t@p add.u32 %0, %0, 4;\n\t}"
            : "+r"(sp)
            : "r"(w), "r"(hibit), "r"(v)
            : "memory");
    else
        asm volatile(
            "{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
            "and.b32 t, %1, %2;\n\tsetp.eq.b32 p, t, 0;\n\t"
            "@p st.shared.u32 [%0], %3;\n\t@p add.u32 %0, %0, 4;\n\t}"
            : "+r"(sp)
            : "r"(w), "r"(hibit), "r"(v)
            : "memory");
}

// ---- fast delta units: odd lane strides ----
//
// Bank conflicts of the staging stores decide these slices' speed: with
// 32-byte lanes, dense data puts the k-th output of every lane 32 words
// apart, i.e. in one bank (the XOR swizzle of decode_range_ll spreads them
// over 8 banks -- still 4-way).  Here a lane takes 4 * kNW - 1 bytes, an odd
// stride, so the k-th outputs of dense lanes fall in distinct banks; the
// staging is plain (no per-store swizzle).  A 4 KiB unit is three 992-byte
// slices of 31-byte lanes and one 1120-byte slice of 35-byte lanes.  Each
// lane reads its bytes and the 4 before them from the unit buffer with
// word loads and funnel shifts; its last word's top byte (the next lane's
// first) is masked out as a digit-0 continuation byte.

// One d3 slice at unit offset `off` (bytes) with lanes of 4 * kNW - 1 bytes.
// Copy-out of a d3 slice: stage[first, end) -> ob[first, end) with ob 16-byte
// aligned (stage[i] <-> ob[i]).  The whole slice lies before the count limit
// (the d3 path's precondition), so nothing is clipped: the whole quads leave
// as one bulk copy, the <= 3 + 3 integers of the partial quads by lanes 0..7
// (stage_out_bulk's protocol, without its 64-bit range arithmetic).
__device__ __forceinline__ void stage_out_d3(uint32_t st_base, uint32_t first, uint32_t end, uint32_t* ob, int lane,
                                             unsigned long long pol) {
    const uint32_t i0 = (first + 3u) & ~3u, i1 = end & ~3u;
    // (the copied range lies in the staging buffer; the bulk copy's ends are 16-byte aligned)
    MVB_CHECK(first <= end && end <= static_cast<uint32_t>(kFStage) && (reinterpret_cast<uintptr_t>(ob) & 15u) == 0u);
#if MVB_OUT_PRED
    // branch-free: every lane computes its (possibly unused) single integer's
    // place -- lanes 0..3 the head quad's [first, i0), lanes 4..7 the tail quad's
    // [i1, end) -- and the copies are predicated instructions
    const uint32_t i = lane < 4 ? (first & ~3u) + static_cast<uint32_t>(lane) : i1 + static_cast<uint32_t>(lane - 4);
    const uint32_t p1 = (lane < 8 && i < end && (lane < 4 ? (i >= first && i < i0) : i >= i0)) ? 1u : 0u;
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
#else
    if (lane < 8) {
        const uint32_t i = lane < 4 ? (first & ~3u) + static_cast<uint32_t>(lane) : i1 + static_cast<uint32_t>(lane - 4);
        if (lane < 4 ? (i >= first && i < i0 && i < end) : (i < end && i >= i0)) {
            uint32_t v;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(st_base + 4u * i) : "memory");
            __stcs(ob + i, v);
        }
    }
    if (lane == 0) {
        if (i1 > i0)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(ob + i0),
                         "r"(st_base + 4u * i0), "r"(4u * (i1 - i0)), "l"(pol)
                         : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
#endif
}

// op (in/out): the slice's first output, out + its index.
// kCheck (batched lists: no totals pass has looked at the bytes): the slice is
// decoded only if no byte of it follows three continuation bytes and all its
// integers end before `lim`; otherwise nothing is stored, op and carry stay,
// and the result is false (the caller takes the general path from the slice
// start).  skip: the slice's first `skip` integers are not stored (a list's
// first slice: the <= 15 bytes before the list in its 16-byte-aligned unit
// are zeroed in shared memory and decode as that many zeros).
// A checked slice whose last integer is integer count-1 (op + its integers ==
// lim) is decoded too; *end_off then receives the slice offset of the byte
// after that integer (otherwise 0).  pad: the slice's last `pad` bytes lie
// past the list's end and are zeroed in shared memory (a list's last slice):
// they decode as that many integers after the real ones -- the first of them
// may close an integer the list leaves unfinished -- which are not stored.
template <int kNW, bool kCheck = false>
__device__ __forceinline__ bool slice_d3_odd(uint32_t ubuf, uint32_t off, uint32_t st_base, uint32_t*& op,
                                             uint32_t& carry, int lane, unsigned long long pol, uint32_t skip = 0u,
                                             const uint32_t* lim = nullptr, uint32_t* end_off = nullptr,
                                             uint32_t pad = 0u) {
    constexpr int kStride = 4 * kNW - 1;
    const uint32_t a = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(op) >> 2) & 3u;  // staging offset of the slice
    // the lane's bytes [b0, b0 + kStride) and the 4 before them
    const uint32_t h0 = ubuf + off + static_cast<uint32_t>(kStride * lane) - 4u;
    const uint32_t sh = 8u * (h0 & 3u);
    const uint32_t wa = h0 & ~3u;
    uint32_t r[kNW + 2];
#pragma unroll
    for (int k = 0; k < kNW + 2; ++k) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r[k]) : "r"(wa + 4u * k) : "memory");
    uint32_t w[kNW + 1];
#pragma unroll
    for (int k = 0; k < kNW + 1; ++k) w[k] = __funnelshift_r(r[k], r[k + 1], sh);
    // w[0]: the 4 bytes before; w[1 .. kNW]: the lane's bytes, the last one the next lane's
    w[kNW] |= 0x80000000u;
    uint32_t W01[kNW], W23[kNW], w7[kNW], tk[kNW];
    uint32_t cp = w[0] & 0x80808080u, cc = 0;
    // kCheck: bit 7 of a byte that ends a run of three continuation bytes
    uint32_t run3 = kCheck ? (cp & (cp << 8) & (cp << 16)) : 0u;
#pragma unroll
    for (int k = 0; k < kNW; ++k) {
        const uint32_t ck = w[k + 1] & 0x80808080u;
        cc = __dp4a(ck, 0x01010101u, cc);  // 128 per continuation byte
        // byte j: 1 if byte j-1 continues, 0x81 if bytes j-1 and j-2 do
        uint32_t x;
        if (kCheck) {
            const uint32_t two = __funnelshift_l(cp, ck, 8) & __funnelshift_l(cp, ck, 16);
            x = __funnelshift_l(cp, ck, 1) | two;
            run3 |= (k == kNW - 1 ? ck & 0x00FFFFFFu : ck) & two;
        } else {
            x = __funnelshift_l(cp, ck, 1) | (__funnelshift_l(cp, ck, 8) & __funnelshift_l(cp, ck, 16));
        }
        W01[k] = prmt_sign(x, 0u, 0x4140u) * 127u + 0x00010001u;
        W23[k] = prmt_sign(x, 0u, 0x4342u) * 127u + 0x00010001u;
        w7[k] = w[k + 1] ^ ck;
        if (k == kNW - 1) w7[k] &= 0x00FFFFFFu;  // (the next lane's byte weighs nothing)
        tk[k] = dp2a_lo(W01[k], w7[k], dp2a_hi(W23[k], w7[k], 0u));
        cp = ck;
    }
    const uint32_t n_own = 4u * kNW - (cc >> 7);
    uint32_t incl = n_own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    const uint32_t n_w = __shfl_sync(0xFFFFFFFFu, incl, 31);
    uint32_t tot = tk[0];
#pragma unroll
    for (int k = 1; k < kNW; ++k) tot += tk[k];
    // kCheck, a slice with integers of 4 or 5 bytes: the weights above count a
    // byte after three (four) continuation bytes as 2^14; a second dp2a chain
    // adds the rest, (2^21 - 2^14) = 127 x 2^14 and (2^28 - 2^14) = 16383 x 2^14
    // (16-bit weights 127 x {1, 129} from a byte code with bit 0 = three
    // continuation bytes before, bit 7 = four).  The tables are rebuilt per
    // word in both passes (lane total, outputs) instead of kept in registers.
    bool lng = false;
    auto long_word = [&](int k, uint32_t& B01, uint32_t& B23, uint32_t& bad) {
        const uint32_t ck = w[k + 1] & 0x80808080u, cq = w[k] & 0x80808080u;
        const uint32_t c3 = __funnelshift_l(cq, ck, 8) & __funnelshift_l(cq, ck, 16) & __funnelshift_l(cq, ck, 24);
        const uint32_t c4 = c3 & cq;  // (byte j of the word before is byte j - 4)
        const uint32_t xb = (c3 >> 7) | c4;
        B01 = prmt_sign(xb, 0u, 0x4140u) * 127u;
        B23 = prmt_sign(xb, 0u, 0x4342u) * 127u;
        // strict mode: a fifth byte must be < 0x10 (internal.hpp:35)
        const uint32_t x = w[k + 1];
        const uint32_t hi4 = x | (x << 1) | (x << 2) | (x << 3);
        bad |= c4 & hi4 & (k == kNW - 1 ? 0x00808080u : 0x80808080u);
    };
    if (kCheck) {
        if (op + (n_w - pad) > lim) return false;
        uint32_t eo = 0;
        if (op + (n_w - pad) == lim) {
            // the byte after the slice's last terminator (before the padding)
            const int vl = static_cast<int>(kStride * 32 - pad) - kStride * lane;  // the lane's bytes before the padding
            uint32_t e = 0;
#pragma unroll
            for (int k = 0; k < kNW; ++k) {
                const uint32_t t = ~w[k + 1] & (k == kNW - 1 ? 0x00808080u : 0x80808080u) & low_bytes_mask(vl - 4 * k);
                if (t) e = 4u * k + ((39u - __clz(t)) >> 3);
            }
            eo = __reduce_max_sync(0xFFFFFFFFu, e ? static_cast<uint32_t>(kStride * lane) + e : 0u);
        }
        *end_off = eo;
        lng = __any_sync(0xFFFFFFFFu, (run3 & 0x80808080u) != 0u);
        if (lng) {
            uint32_t tb = 0, bad = 0;
#pragma unroll
            for (int k = 0; k < kNW; ++k) {
                uint32_t B01, B23;
                long_word(k, B01, B23, bad);
                tb = dp2a_lo(B01, w7[k], dp2a_hi(B23, w7[k], tb));
            }
            if (__any_sync(0xFFFFFFFFu, bad != 0u)) return false;  // malformed: the general path reports it
            tot += tb << 14;
        }
    }
    uint32_t acc = lane_scan_offset<true>(tot, carry);
    uint32_t sp = st_base + 4u * (a + incl - n_own);
    MVB_CHECK(a + n_w <= static_cast<uint32_t>(kFStage));
#if MVB_BULK_OUT
    stage_wait_read(lane);  // the previous slice's copy-out has read the staging buffer
    __syncwarp();
#endif
    if (kCheck && lng) {
        uint32_t accb = 0;
#pragma unroll
        for (int k = 0; k < kNW; ++k) {
            uint32_t B01, B23, bad = 0;
            long_word(k, B01, B23, bad);
            const uint32_t o0 = dp2a_lo(W01[k] & 0xFFFFu, w7[k], acc);
            const uint32_t o1 = dp2a_lo(W01[k], w7[k], acc);
            const uint32_t o2 = dp2a_hi(W23[k] & 0xFFFFu, w7[k], o1);
            acc += tk[k];
            const uint32_t b0 = dp2a_lo(B01 & 0xFFFFu, w7[k], accb);
            const uint32_t b1 = dp2a_lo(B01, w7[k], accb);
            const uint32_t b2 = dp2a_hi(B23 & 0xFFFFu, w7[k], b1);
            accb = dp2a_hi(B23, w7[k], b1);
            slot_store_w<false>(sp, w[k + 1], 0x80u, o0 + (b0 << 14));
            slot_store_w<false>(sp, w[k + 1], 0x8000u, o1 + (b1 << 14));
            slot_store_w<false>(sp, w[k + 1], 0x800000u, o2 + (b2 << 14));
            slot_store_w<false>(sp, w[k + 1], 0x80000000u, acc + (accb << 14));
        }
    } else {
#pragma unroll
        for (int k = 0; k < kNW; ++k) {
            const uint32_t o0 = dp2a_lo(W01[k] & 0xFFFFu, w7[k], acc);
            const uint32_t o1 = dp2a_lo(W01[k], w7[k], acc);
            const uint32_t o2 = dp2a_hi(W23[k] & 0xFFFFu, w7[k], o1);
            acc += tk[k];
            slot_store_w<false>(sp, w[k + 1], 0x80u, o0);
            slot_store_w<false>(sp, w[k + 1], 0x8000u, o1);
            slot_store_w<false>(sp, w[k + 1], 0x800000u, o2);
            slot_store_w<false>(sp, w[k + 1], 0x80000000u, acc);
        }
    }
#if MVB_BULK_OUT
    stage_fence();
    __syncwarp();
    MVB_CHECK(sp <= st_base + 4u * (a + incl));  // (each lane stored exactly its own integers)
    stage_out_d3(st_base, a + skip, a + n_w - pad, op - a, lane, pol);
    op += n_w - pad;
#else
    __syncwarp();
    MVB_CHECK(sp <= st_base + 4u * (a + incl));  // (each lane stored exactly its own integers)
    if (n_w - pad > skip)
        stage_out<false>(st_base + 4u * ((a + skip) & ~3u), (a + skip) & 3u, n_w - pad - skip, (a + skip) & 3u, ~0ull,
                         op - a + ((a + skip) & ~3u), lane);
    op += n_w - pad;
    __syncwarp();  // the staging buffer is rewritten by the next slice
#endif
    return true;
}

// A delta unit staged in shared memory whose integers all have at most 3
// bytes, with integer limit-1 outside it (both known from its totals pass):
// every slice takes the dp2a path with no range masks, votes or limit checks.
// carry: every byte before the unit (the prefix tree's sums count bytes, so
// no straddle correction); values go to out[base ...].
// op: the unit's first output (out + its index).
__device__ __forceinline__ void decode_unit_d3(uint32_t ubuf, uint32_t* op, uint32_t carry, uint32_t st_base, int lane,
                                               unsigned long long pol) {
    static_assert(kUnit == 3 * 992 + 1120, "the d3 slicing covers a 4 KiB unit");
#pragma unroll 1
    for (int i = 0; i < 3; ++i) (void)slice_d3_odd<8>(ubuf, 992u * i, st_base, op, carry, lane, pol);
    (void)slice_d3_odd<9>(ubuf, 2976u, st_base, op, carry, lane, pol);
}

// A staged unit whose integers all have the same length L = 4 or 5 (sparse
// streams: hashed ids, the all-5-byte point of BASELINE config 5 -- the
// reference has a window kernel for just this shape, two5b_lanes,
// decode_simd.cpp:68-79).  The terminators of such a unit form an arithmetic
// progression, so integer j ends at byte e0 + L * j: instead of 32 byte slots
// per lane (6 of them used), lane l assembles integers l, l + 32, ... -- two
// ld.shared, a funnel shift, two dp4a -- and stores them straight to global
// memory, consecutive lanes to consecutive integers (no staging).  Delta: one
// warp scan per pass of 32 integers.
//   ubuf: the unit in shared memory (the 16 bytes before it too); n_ints: its
//   integers (the totals pass's count), all before the count limit; op: their
//   place in the output; carry (delta): the value before the unit's first
//   integer (complete integers only).
// False -- nothing decided, the caller takes another path -- if the unit is not
// of this shape, or (strict mode, internal.hpp:35) a fifth byte is >= 0x10;
// what was stored until then is what the general path stores again.
template <bool kDelta>
__device__ __noinline__ bool unit_uniform(uint32_t ubuf, uint32_t n_ints, uint32_t* op, uint32_t carry) {
    const int lane = threadIdx.x & 31;
    // the first two terminators of the unit (in lane 0's 32 bytes): e0 and L
    uint32_t T[kUnit / kLLSlice];
#pragma unroll
    for (int i = 0; i < kUnit / kLLSlice; ++i) {
        const uint32_t sa = ubuf + static_cast<uint32_t>(kLLSlice * i + 32 * lane);
        const uint4 x0 = lds128(sa), x1 = lds128(sa + 16u);
        T[i] = hibits16(~x0.x, ~x0.y, ~x0.z, ~x0.w) | (hibits16(~x1.x, ~x1.y, ~x1.z, ~x1.w) << 16);
    }
    const uint32_t t0 = __shfl_sync(0xFFFFFFFFu, T[0], 0);
    const uint32_t t1 = t0 & (t0 - 1u);
    if (t1 == 0u) return false;
    const uint32_t e0 = __ffs(t0) - 1u, L = (__ffs(t1) - 1u) - e0;
    if (L < 4u || L > 5u || e0 >= L) return false;
    // the integer ending at e0 has L bytes too: a terminator (or the stream's start,
    // zeros) at e0 - L, continuation bytes after it
    bool ok = true;
    if (lane < 5) {
        const int pos = static_cast<int>(e0) - static_cast<int>(L) + lane;  // e0 - L .. e0 - L + 4
        if (pos < 0) {
            uint32_t b;
            asm volatile("ld.shared.u8 %0, [%1];" : "=r"(b) : "r"(ubuf + pos) : "memory");
            ok = lane == 0 ? b < 0x80u : b >= 0x80u;
        }
    }
    // every lane's terminators are the progression's: bits r + k L of each 32-byte word
    const uint32_t pat = L == 5u ? 0x42108421u : 0x11111111u;
    uint32_t r = (e0 + L * 1024u - 32u * static_cast<uint32_t>(lane)) % L;  // first expected position in slice 0's lane bytes
    const uint32_t step = L - (static_cast<uint32_t>(kLLSlice) % L);        // the same for the next slice: + step (mod L)
#pragma unroll
    for (int i = 0; i < kUnit / kLLSlice; ++i) {
        ok = ok && T[i] == (pat << r);
        r += step;
        if (r >= L) r -= L;
    }
    const uint32_t n = (static_cast<uint32_t>(kUnit) - 1u - e0) / L + 1u;
    if (!__all_sync(0xFFFFFFFFu, ok) || n != n_ints) return false;
    // the gather: four passes of 32 integers per iteration, independent of one
    // another (their shared-memory loads and, delta, their warp scans overlap)
    constexpr int kQ = 4;
    uint32_t bad = 0;
    const uint32_t sh = 28u - 7u * L;  // (L = 4: 0)
#pragma unroll 1
    for (uint32_t j0 = 0; j0 < n; j0 += 32u * kQ) {
        uint32_t v[kQ];
        bool act[kQ];
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            const uint32_t j = j0 + 32u * q + static_cast<uint32_t>(lane);
            act[q] = j < n;
            // the integer's last byte (past the end: another integer's).  (The plain and the
            // delta instantiation each keep the form that measured faster: all-5B plain 192
            // vs 410 us with the delta form, delta 295 vs 311 us with the plain form.)
            const uint32_t a = ubuf + e0 + L * (kDelta ? (j < n ? j : n - 1u) : (act[q] ? j : 0u));
            uint32_t lo, hi;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(lo) : "r"((a & ~3u) - 4u) : "memory");
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(hi) : "r"(a & ~3u) : "memory");
            const uint32_t t = a & 3u;
            const uint32_t x = __funnelshift_rc(lo, hi, 8u * t + 8u);  // bytes a - 3 .. a (t = 3: hi itself)
            uint32_t w = pack28(x);
            if (L == 5u) {
                w = (w << 7) | ((lo >> (8u * t)) & 0x7Fu);  // the first byte: byte t of lo
                // the fifth byte's bits 4..6 (bit 7: a terminator)
                if (kDelta) bad |= x & 0x70000000u;
                else bad |= act[q] ? (x >> 28) & 7u : 0u;
            } else {
                w >>= sh;
            }
            v[q] = (act[q] || !kDelta) ? w : 0u;
        }
        if (kDelta) {
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
                for (int q = 0; q < kQ; ++q) {
                    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, v[q], o);
                    if (lane >= o) v[q] += y;
                }
            }
#pragma unroll
            for (int q = 0; q < kQ; ++q) {
                v[q] += carry;
                carry = __shfl_sync(0xFFFFFFFFu, v[q], 31);
            }
        }
#pragma unroll
        for (int q = 0; q < kQ; ++q)
            if (act[q]) __stcs(op + j0 + 32u * q + lane, v[q]);
    }
    return !__any_sync(0xFFFFFFFFu, bad != 0u);
}

// A staged delta unit with integers of 4 or 5 bytes (its integers all end
// before lim): checked slices, a second dp2a chain where the long integers
// are.  False if a slice holds a malformed integer (the caller then decodes
// the unit again with the general path, which reports it; the slices stored so
// far are what it stores).
__device__ __noinline__ bool unit_d3_checked(uint32_t ubuf, uint32_t* op, uint32_t carry, uint32_t st_base,
                                             const uint32_t* lim, unsigned long long pol) {
    const int lane = threadIdx.x & 31;
    uint32_t eo;
#pragma unroll 1
    for (int i = 0; i < 3; ++i)
        if (!slice_d3_odd<8, true>(ubuf, 992u * i, st_base, op, carry, lane, pol, 0u, lim, &eo)) return false;
    return slice_d3_odd<9, true>(ubuf, 2976u, st_base, op, carry, lane, pol, 0u, lim, &eo);
}

// decode_range_ll's per-slice algorithm over the unit [qs, qe) staged in
// shared memory at ubuf (byte qs; the 16 bytes before it too), or -- ubuf 0,
// units at the stream's edges -- read from global memory with range masks.
// kIn: the unit is staged, lies inside the stream with the 16 bytes before it,
// and all its integers end before `limit` -- every slice is interior, nothing
// is masked or clipped, no slice holds integer limit-1 (plain streams' common
// units: the range logic below was a fifth of c1's instructions).
template <bool kDelta, bool kSwz, bool kIn = false>
__device__ __forceinline__ void decode_unit_ll(const ByteRange& R, long long qs, long long qe,
                                                unsigned long long base, uint32_t carry, unsigned long long limit,
                                                uint32_t* out, uint32_t* stage, uint32_t ubuf, int lane,
                                                const RangeSink& K, RangeOut& ro, unsigned long long pol) {
    const uint32_t out_w = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(out) >> 2);
    const uint32_t st_base = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
    const int ns = kIn ? kUnit / kLLSlice : static_cast<int>((qe - qs + kLLSlice - 1) / kLLSlice);
    int i_lo = 0, i_hi = ns;  // interior slices: i_lo <= i < i_hi
    if (!kIn) {
        const long long d = R.lo - qs, e = R.hi - qs;
        const long long lo = d <= 0 ? 0 : (d + kLLSlice - 1) / kLLSlice;
        const long long hi = e <= 0 ? 0 : e / kLLSlice;
        i_lo = static_cast<int>(lo < ns ? lo : ns);
        i_hi = static_cast<int>(hi < ns ? hi : ns);
    }
    unsigned long long run = base;  // output index of the slice's first integer
    int last_i = -1;                // the last slice holding an integer (warp-uniform)
    uint32_t pw2 = 0, pw3 = 0;      // lane 0: the 8 bytes before the slice
    if (lane == 0) {
        if (ubuf) {
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(pw2), "=r"(pw3) : "r"(ubuf - 8u) : "memory");
        } else if (r_inside(R, qs - 8, 8)) {
            const uint2 v = __ldg(reinterpret_cast<const uint2*>(R.ab + qs - 8));
            pw2 = v.x;
            pw3 = v.y;
        } else {
            pw2 = r_word(R, qs - 8);
            pw3 = r_word(R, qs - 4);
        }
    }
#pragma unroll 1
    for (int i = 0; i < ns; ++i) {
        const uint32_t a = (out_w + static_cast<uint32_t>(run)) & 3u;  // staging offset of the slice
        const bool inter = kIn || (i >= i_lo && i < i_hi);             // warp-uniform
        const long long q0 = qs + static_cast<long long>(kLLSlice) * i + 32 * lane;
        uint4 x0, x1;
        if (kIn || (inter && ubuf)) {
            const uint32_t sa = ubuf + static_cast<uint32_t>(kLLSlice * i + 32 * lane);
            x0 = lds128(sa);
            x1 = lds128(sa + 16u);
        } else {
            x0 = r_load16(R, q0);
            x1 = r_load16(R, q0 + 16);
        }
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
        // delta: no byte after three continuation bytes in positions 0..31 (every
        // integer ending here has at most 3 bytes) -> the dp2a path
        bool take3 = false;
        if (kDelta) {
            const unsigned long long t3 = C & (C >> 1) & (C >> 2) & 0x1FFFFFFFEull;
            take3 = (inter || tail || MVB_HEAD2) && !__any_sync(0xFFFFFFFFu, t3 != 0);
        }
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
#if MVB_BULK_OUT
        stage_wait_read(lane);  // an earlier copy-out (this unit's or the previous one's) has read the staging buffer
        __syncwarp();
#endif
        if (take3) {
            // carry: complete integers before the slice -> every byte before it
            const uint32_t hin = __shfl_sync(0xFFFFFFFFu, tail_value(wp3), 0);
            const uint32_t hout = __shfl_sync(0xFFFFFFFFu, tail_value(w[7]), 31);
            carry += hin;
            lane_slots_d3<kSwz>(wp3, w, T32 & inr32, st_base + 4u * (a + wexcl), carry);
            carry -= hout;
            if (!kIn && run < limit && run + n_w >= limit)
                slice_count_end(R, K, q0, T32 & inr32, static_cast<uint32_t>(limit - 1 - run), wexcl, n_own);
        } else if (take2 || takef || takef5) {
            if (take2)
                lane_slots_2b<kDelta, kSwz, 8>(wp3, w, T32 & inr32, st_base + 4u * (a + wexcl), carry);
            else if (!kDelta && takef5)
                lane_slots_fast<kDelta, kSwz, true>(wp3, w, T32, st_base + 4u * (a + wexcl), carry, F5);
            else
                lane_slots_fast<kDelta, kSwz>(wp3, w, T32, st_base + 4u * (a + wexcl), carry);
            // the slice holds integer limit-1: record its end (stores past limit are
            // dropped by the copy-out)
            if (!kIn && run < limit && run + n_w >= limit)
                slice_count_end(R, K, q0, T32 & inr32, static_cast<uint32_t>(limit - 1 - run), wexcl, n_own);
        } else
            carry = ll_slice_gen<kDelta, kSwz>(R, q0, x0, x1, wp2, wp3, T32, inr32, n_w, wexcl, run, limit, K,
                                               st_base + 4u * (a + wexcl), st_base + kSparseWin + 72u * lane, carry);
        if (n_w == 0) continue;
#if MVB_BULK_OUT
        if (!kSwz) {
            stage_fence();
            __syncwarp();
            if (kIn) stage_out_d3(st_base, a, a + n_w, out + run - a, lane, pol);
            else stage_out_bulk(st_base, a, n_w, run, limit, out, lane, pol);
            run += n_w;
            continue;
        }
#endif
        __syncwarp();
        stage_out<kSwz>(st_base, a, n_w, run, kIn ? ~0ull : limit, out, lane);
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

__device__ __forceinline__ void fentry_put(FEntry* e, unsigned long long cnt, uint32_t sum, unsigned tag,
                                           uint32_t flags = 0u) {
    // (bits 24..31 of the sum word: a unit's totals-pass flags, level 0 only)
    const ulonglong2 v = make_ulonglong2((cnt << 24) | tag,
                                         (static_cast<unsigned long long>(sum) << 32) | ((flags & 0xFFu) << 24) | tag);
    asm volatile("st.global.cg.v2.u64 [%0], {%1, %2};" ::"l"(e), "l"(v.x), "l"(v.y) : "memory");
}
// Wait for entry e of this launch (tag) and return its count and sum.
__device__ __forceinline__ void fentry_get(const FEntry* e, unsigned tag, unsigned long long& cnt, uint32_t& sum) {
    unsigned long long c, s;
    for (;;) {
        asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(c), "=l"(s) : "l"(e) : "memory");
        if ((c & 0xFFFFFFull) == tag && (s & 0xFFFFFFull) == tag) break;
        __nanosleep(MVB_F_SLEEP);
    }
    cnt = c >> 24;
    sum = static_cast<uint32_t>(s >> 32);
}

// Publish entry i of level l (one lane) and aggregate upwards: the last
// child to arrive at a parent sums the parent's children (the whole warp).
__device__ __forceinline__ void fused_publish(const FusedParams& F, int l, uint32_t i, unsigned long long cnt,
                                              uint32_t sum, unsigned tag, int lane, uint32_t flags = 0u) {
    for (;;) {
        if (lane == 0) fentry_put(F.tree[l] + i, cnt, sum, tag, l == 0 ? flags : 0u);
        if (l + 1 >= F.levels) return;
        const uint32_t par = i >> 5;
        const uint32_t left = static_cast<uint32_t>(F.n_at[l]) - (par << 5);  // children from the parent's first on
        unsigned last = 0;
        if (lane == 0) {
            const unsigned n = atomicAdd(F.arrive[l + 1] + par, 1u) + 1u;
            if (left >= 32u) last = (n & 31u) == 0u ? 1u : 0u;
            else last = n % left == 0u ? 1u : 0u;  // (the level's last, partial parent)
        }
        last = __shfl_sync(0xFFFFFFFFu, last, 0);
        if (!last) return;
        const uint32_t kids = left < 32u ? left : 32u;
        unsigned long long c = 0;
        uint32_t s = 0;
        if (static_cast<uint32_t>(lane) < kids) fentry_get(F.tree[l] + ((par << 5) + lane), tag, c, s);
        sum = __reduce_add_sync(0xFFFFFFFFu, s);
        if (F.narrow) {
            cnt = __reduce_add_sync(0xFFFFFFFFu, static_cast<uint32_t>(c));
        } else {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
            cnt = c;
        }
        i = par;
        ++l;
    }
}

// Sum of the entries before index v at every level (all lanes get it): the
// count and value sum of segments [0, v).  Waits for entries not yet
// published in this launch.
__device__ __forceinline__ void fused_prefix(const FusedParams& F, long long v, unsigned tag, int lane,
                                             unsigned long long& cnt, unsigned long long& sum) {
    unsigned long long c = 0;
    uint32_t s = 0;
    for (int l = 0; l < F.levels; ++l) {
        const long long d = (v >> (5 * l)) & 31;
        if (lane < d) {
            unsigned long long ec;
            uint32_t es;
            fentry_get(F.tree[l] + (((v >> (5 * l)) >> 5) << 5) + lane, tag, ec, es);
            c += ec;
            s += es;
        }
    }
    sum = __reduce_add_sync(0xFFFFFFFFu, s);
    if (F.narrow) {
        cnt = __reduce_add_sync(0xFFFFFFFFu, static_cast<uint32_t>(c));
    } else {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
        cnt = c;
    }
}

// fused_totals for a unit staged in shared memory (ubuf: its first byte; the
// 16 bytes before it are there too): n_it 1 KiB iterations, all inside the
// stream -- no range masks, 32-bit addressing.
// kLong (the long-integer instantiations): an iteration with integers of 4+
// bytes adds the second chain's correction to the cheap weights -- a byte after
// three (four) continuation bytes was counted as 2^14: (2^21 - 2^14) = 127 x
// 2^14 and (2^28 - 2^14) = (127 + 16256) x 2^14 more, two dp4a over 0/1 class
// flags -- instead of recomputing every weight exactly.
template <bool kDelta, bool kLong = false>
__device__ __forceinline__ void unit_totals(uint32_t ubuf, int n_it, int lane, unsigned& cnt_out, uint32_t& sum_out,
                                            uint32_t& flags_out) {
    uint32_t h1 = 0;  // lane 0: the word before the iteration
    if (lane == 0) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(h1) : "r"(ubuf - 4u) : "memory");
    uint32_t cc = 0, sA = 0, sB = 0, sX = 0, flags = 0;
#pragma unroll 1
    for (int it = 0; it < n_it; ++it) {
        const uint32_t sa = ubuf + static_cast<uint32_t>(kLLSlice * it + 32 * lane);
        const uint4 x0 = lds128(sa), x1 = lds128(sa + 16u);
        const uint32_t w[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        uint32_t p1 = __shfl_up_sync(0xFFFFFFFFu, w[7], 1);
        const uint32_t l1 = __shfl_sync(0xFFFFFFFFu, w[7], 31);
        if (lane == 0) p1 = h1;
        h1 = l1;
        if (kDelta) {
            uint32_t hi3 = 0, a = 0, b = 0;
            ftot_word(w[0], p1, cc, a, b, hi3);
#pragma unroll
            for (int k = 1; k < 8; ++k) ftot_word(w[k], w[k - 1], cc, a, b, hi3);
            if (kLong && __any_sync(0xFFFFFFFFu, hi3 != 0)) {
                flags |= 1u;
                uint32_t x3 = 0, x4 = 0;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t ck = w[k] & 0x80808080u, cq = (k ? w[k - 1] : p1) & 0x80808080u;
                    const uint32_t c3 = __funnelshift_l(cq, ck, 1) & __funnelshift_l(cq, ck, 9) & __funnelshift_l(cq, ck, 17);
                    const uint32_t c4 = c3 & (cq >> 7);  // (byte j of the word before is byte j - 4)
                    const uint32_t w7 = w[k] ^ ck;
                    x3 = __dp4a(w7, c3, x3);
                    x4 = __dp4a(w7, c4, x4);
                }
                sA += a;
                sB += b;
                sX += (127u * x3 + 16256u * x4) << 14;
            } else if (__any_sync(0xFFFFFFFFu, hi3 != 0)) {  // an integer of 4+ bytes: the exact weights
                flags |= 1u;
                uint32_t p2 = __shfl_up_sync(0xFFFFFFFFu, w[6], 1);
                if (lane == 0) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(p2) : "r"(sa - 8u) : "memory");
                uint32_t x = ftot_word_exact(w[0], p1, p2) + ftot_word_exact(w[1], w[0], p1);
#pragma unroll
                for (int k = 2; k < 8; ++k) x += ftot_word_exact(w[k], w[k - 1], w[k - 2]);
                sX += x;
            } else {
                sA += a;
                sB += b;
            }
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) cc = __dp4a(w[k] & 0x80808080u, 0x01010101u, cc);
        }
    }
    flags_out = flags;
    cnt_out = __reduce_add_sync(0xFFFFFFFFu, 32u * static_cast<unsigned>(n_it) - (cc >> 7));
    sum_out = kDelta ? __reduce_add_sync(0xFFFFFFFFu, sA + (sB << 14) + sX) : 0u;
}

// fused_prefix in two halves: the entries' loads are issued early (their
// latency overlaps other work), the tags checked -- and stale entries
// waited for -- later.  v < n_seg <= 32^levels, so v >> (5 * l) is 0 at the
// levels not in use: they cost a shift and a compare.
struct PrefixLoads {
    unsigned long long c[kFLevels], s[kFLevels];
};
__device__ __forceinline__ void fused_prefix_issue(const FusedParams& F, uint32_t v, int lane, PrefixLoads& P) {
#pragma unroll
    for (int l = 0; l < kFLevels; ++l) {
        const uint32_t vl = v >> (5 * l);
        if (static_cast<uint32_t>(lane) < (vl & 31u)) {
            const FEntry* e = F.tree[l] + ((vl & ~31u) + static_cast<uint32_t>(lane));
            asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(P.c[l]), "=l"(P.s[l]) : "l"(e) : "memory");
        }
    }
}
template <bool kNarrow>
__device__ __forceinline__ void fused_prefix_finish_n(const FusedParams& F, uint32_t v, unsigned tag, int lane,
                                                      PrefixLoads& P, unsigned long long& cnt, uint32_t& sum) {
    unsigned long long c = 0;
    uint32_t c32 = 0, s = 0;
#pragma unroll
    for (int l = 0; l < kFLevels; ++l) {
        const uint32_t vl = v >> (5 * l);
        if (static_cast<uint32_t>(lane) < (vl & 31u)) {
            unsigned long long pc = P.c[l], ps = P.s[l];
            while ((static_cast<uint32_t>(pc) & 0xFFFFFFu) != tag || (static_cast<uint32_t>(ps) & 0xFFFFFFu) != tag) {
                __nanosleep(MVB_F_SLEEP);
                const FEntry* e = F.tree[l] + ((vl & ~31u) + static_cast<uint32_t>(lane));
                asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(pc), "=l"(ps) : "l"(e) : "memory");
            }
            if (kNarrow) c32 += static_cast<uint32_t>(pc >> 24);
            else c += pc >> 24;
            s += static_cast<uint32_t>(ps >> 32);
        }
    }
    sum = __reduce_add_sync(0xFFFFFFFFu, s);
    if (kNarrow) {
        cnt = __reduce_add_sync(0xFFFFFFFFu, c32);
    } else {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
        cnt = c;
    }
}
__device__ __forceinline__ void fused_prefix_finish(const FusedParams& F, uint32_t v, unsigned tag, int lane,
                                                    PrefixLoads& P, unsigned long long& cnt, uint32_t& sum) {
    if (F.narrow) fused_prefix_finish_n<true>(F, v, tag, lane, P, cnt, sum);
    else fused_prefix_finish_n<false>(F, v, tag, lane, P, cnt, sum);
}

// Completion (all threads of every CTA): the last CTA produces the DecodeResult.
__device__ __forceinline__ void fused_complete(const FusedParams& F, unsigned tag) {
    const SegParams& S = F.S;
    __shared__ bool s_last;
    __shared__ long long s_seg;
    __shared__ unsigned long long s_total;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&S.hdr->done, 1ull) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x < 32) {
        unsigned long long c, u;
        fused_prefix(F, S.n_seg, tag, threadIdx.x, c, u);
        if (threadIdx.x == 0) {
            s_total = c;
            if (F.mode == 1) {  // a totals pass: the record, no DecodeResult
                F.rec[0] = c;
                F.rec[1] = u & 0xFFFFFFFFull;
            }
        }
    }
    __syncthreads();
    const unsigned long long total = s_total;
    WsHeader* h = S.hdr;
    if (F.mode == 1) {
        if (threadIdx.x == 0) {
            h->done = 0;
            h->ticket = 0;
            h->epoch = h->epoch + 1;
        }
        __threadfence();
        return;
    }
    const unsigned long long err_inv = *reinterpret_cast<volatile unsigned long long*>(&h->err_idx_inv);
    const bool truncated = !(err_inv != 0ull && ~err_inv < S.count) && total < S.count;  // (CTA-uniform)
    long long last_end_found = 0;
    if (truncated) {
        // the end of the stream's last integer: the last segment holding one,
        // then its last terminator byte
        if (threadIdx.x == 0) s_seg = -1;
        __syncthreads();
        for (long long hi = S.n_seg - 1; hi >= 0; hi -= blockDim.x) {
            const long long k = hi - static_cast<long long>(threadIdx.x);
            if (k >= 0 && (__ldcg(&F.tree[0][k].c) >> 24) > 0) atomicMax(&s_seg, k);
            __syncthreads();
            if (s_seg >= 0) break;
        }
        if (s_seg >= 0) {
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
    if (threadIdx.x == 0) {
        const unsigned long long errpos_inv = *reinterpret_cast<volatile unsigned long long*>(&h->err_pos_inv);
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
            r.bytes_consumed = static_cast<unsigned long long>(last_end_found);
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

__device__ __forceinline__ void mbar_init_warp(unsigned long long* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
// One TMA bulk copy of `bytes` (multiple of 16, 16-byte-aligned ends) into
// shared memory, completing on the mbarrier (issued by one lane).
__device__ __forceinline__ void tma_bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of dst come first
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// Timeline build (-DMVB_F_TRACE=1, scripts/r2/trace_fused.py): every warp
// appends (globaltimer, code) pairs to its 64-entry row of g_ftrace.
#ifndef MVB_F_TRACE
#define MVB_F_TRACE 0
#endif
#if MVB_F_TRACE
__device__ unsigned long long* g_ftrace;
#define MVB_FT(code)                                                                                    \
    do {                                                                                                \
        if (lane == 0 && g_ftrace) {                                                                    \
            unsigned long long* row = g_ftrace + 64ull * (blockIdx.x * kSegWarps + wid);                \
            unsigned long long t_;                                                                      \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                      \
            const unsigned long long n_ = row[0];                                                       \
            if (n_ < 62) {                                                                              \
                row[1 + n_] = (t_ << 4) | (code);                                                       \
                row[0] = n_ + 1;                                                                        \
            }                                                                                           \
        }                                                                                               \
    } while (0)
#else
#define MVB_FT(code) ((void)0)
#endif

// kMode: 0 totals and decode, 1 totals only, 2 decode only (F.mode == kMode;
// separate instantiations keep the common one free of the others' code)
// kStatic0 (mode 0, streams of few units per warp): the first round of units
// is handed out without tickets (a separate instantiation: the long streams'
// kernel stays as it is).
// kLong (delta streams asked for at 2.5+ bytes per integer, plain ones at 4+):
// units of equally long 4- or 5-byte integers take the per-integer gather
// (unit_uniform), other delta units with integers of 4 or 5 bytes checked dp2a
// slices, instead of the general path (a separate instantiation as well:
// hooked into the common kernel, the extra call cost c4 4%).
template <bool kDelta, int kMode, bool kStatic0 = false, bool kLong = false>
__global__ void __launch_bounds__(kSegThreads, kFBlocks) vbyte_fused_decode(const __grid_constant__ FusedParams F) {
    extern __shared__ __align__(128) uint8_t smem[];
    const SegParams& S = F.S;
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    uint8_t* const wbuf = smem + wid * kFWarpBytes;  // two unit buffers: [0, 16) the bytes before, then the unit
    uint32_t* const stage = reinterpret_cast<uint32_t*>(wbuf + 2 * kUnitBuf);
    unsigned long long* const bar_p = reinterpret_cast<unsigned long long*>(smem + kSegWarps * kFWarpBytes) + 2 * wid;
    const uint32_t bar0 = static_cast<uint32_t>(__cvta_generic_to_shared(bar_p));
    const uint32_t buf0 = static_cast<uint32_t>(__cvta_generic_to_shared(wbuf));
    if (lane == 0) {
        mbar_init_warp(bar_p);
        mbar_init_warp(bar_p + 1);
    }
    __syncwarp();
    uint32_t phases = 0;  // bit b: parity of buffer b's next completion
    MVB_FT(1);
    const ByteRange R = {S.in - S.mis, S.mis, S.mis + S.len, S.mis, S.mis + S.len};
    const long long q_stream_end = (R.hi + 15) & ~15ll;
    const RangeSink K = {S.hdr, nullptr, nullptr, nullptr};
    const unsigned long long pol = l2_evict_first();  // (output copies: written once, never read here)
#if MVB_F_PF0
    // While the previous grid on the stream drains: L2 prefetches of the units
    // the first MVB_F_PF0 rounds of tickets will hand out (whichever warps take
    // them).  Only prefetches may come before the wait -- L2 stays coherent with
    // whatever still writes the input; a load into shared memory could be stale.
    if (kMode != 1 && lane == 0) {
        const long long w_all = static_cast<long long>(gridDim.x) * kSegWarps;
#pragma unroll
        for (int r = 0; r < MVB_F_PF0; ++r) {
            const long long q = ((blockIdx.x * kSegWarps + wid) + r * w_all) * kUnit;
            if (q - 16 >= R.lo && q + kUnit <= R.hi)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(R.ab + q), "r"(static_cast<uint32_t>(kUnit))
                             : "memory");
        }
    }
#endif
    // the previous grid on the stream (e.g. the previous decode on this
    // workspace: it resets the ticket and advances the epoch) is complete and
    // visible after this
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    MVB_FT(2);
    // this launch's tree tag; a decode-only launch reads the tree its totals
    // launch (the previous one on this workspace) tagged
    const unsigned long long epoch = *reinterpret_cast<volatile unsigned long long*>(&S.hdr->epoch);
    const unsigned tag = static_cast<unsigned>(kMode == 2 ? epoch : epoch + 1ull) & 0xFFFFFFu;
    const uint32_t prev0 = kDelta ? (S.prev_dev ? S.prev + *S.prev_dev : S.prev) : 0u;
    const uint32_t st_base = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
    // units [u_first, u_end) are staged in shared memory by the TMA: the unit and
    // the 16 bytes before it lie inside the stream
    // (unit 0 of a 16-byte-aligned stream is staged too: nothing lies before it, its
    // 16 bytes before are zeroed in shared memory -- the stream's start is an
    // integer boundary)
    const uint32_t u_end = static_cast<uint32_t>(R.hi / kUnit);
    const uint32_t u_first = R.lo == 0 ? 0u : static_cast<uint32_t>((R.lo + 16 + kUnit - 1) / kUnit);
    const uint32_t n_units = static_cast<uint32_t>(S.n_seg);
    // the stream's last, partial unit is staged as well (whole 16-byte blocks by the
    // TMA, the last bytes one per lane, zeros after them): its totals pass and the
    // whole slices of its decode read shared memory like any other unit's.  Left
    // to masked global loads it was the decode's tail: 7.7 + 15.5 us of one warp
    // on c2, a third of the launch.
    const uint32_t part_bytes = static_cast<uint32_t>(R.hi - static_cast<long long>(u_end) * kUnit);
    const uint32_t u_part = (part_bytes != 0u && u_end >= 1u) ? u_end : 0xFFFFFFFFu;
    unsigned* const ticket = reinterpret_cast<unsigned*>(&S.hdr->ticket);  // (units < 2^28: the low word)
#if MVB_F_PF
    const uint32_t pf_dist = MVB_F_PF * gridDim.x * kSegWarps / 8u;
#endif
    // a delta unit whose integers all have at most 3 bytes (its totals pass's
    // flags), staged, with integer count-1 ending after it: the dp2a path
    auto unit_is_d3 = [&](uint32_t up, unsigned long long base, unsigned c_up, uint32_t f_up) -> bool {
        return kDelta && up >= u_first && up < u_end && !(f_up & 1u) && base + c_up < S.count;
    };
    // (kLong) unit_uniform with the general path's carry: the sum of the complete integers before the unit
    auto unit_uniform_at = [&](uint32_t ubuf, unsigned c_up, uint32_t* op, uint32_t csum) -> bool {
        uint32_t carry = 0;
        if (kDelta) {
            uint32_t wb;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(wb) : "r"(ubuf - 4u) : "memory");
            carry = csum - tail_value(wb) + prev0;
        }
#if MVB_BULK_OUT
        stage_wait_read(lane);  // (no staging here, but a later general fallback rewrites the buffer)
#endif
        return unit_uniform<kDelta>(ubuf, c_up, op, carry);
    };
    // decode unit `up` (buffer bp), given its prefix and its totals pass's count / flags
    auto decode_unit = [&](uint32_t up, int bp, unsigned long long base, uint32_t csum, unsigned c_up, uint32_t f_up) {
        if (base < S.count) {  // (warp-uniform; otherwise nothing of unit up is stored)
            const long long qs = static_cast<long long>(up) * kUnit;
            const long long qe = qs + kUnit < q_stream_end ? qs + kUnit : q_stream_end;
            const bool staged = (up >= u_first && up < u_end) || up == u_part;  // (warp-uniform)
            const uint32_t ubuf = staged ? buf0 + bp * kUnitBuf + 16u : 0u;
            if (unit_is_d3(up, base, c_up, f_up)) {
                // (carry: every byte before the unit)
                uint32_t carry = csum + prev0;
                uint32_t* op = S.out + base;
                decode_unit_d3(ubuf, op, carry, st_base, lane, pol);
            } else if (kLong && up >= u_first && up < u_end && base + c_up < S.count && 7u * c_up <= 2u * kUnit &&
                       unit_uniform_at(ubuf, c_up, S.out + base, csum)) {
                // (kLong: a unit of equally long 4- or 5-byte integers took the gather)
            } else if (kLong && kDelta && up >= u_first && up < u_end && base + c_up < S.count &&
                       unit_d3_checked(ubuf, S.out + base, csum + prev0, st_base, S.out + S.count, pol)) {
                // (kLong: a unit with integers of 4 or 5 bytes took the checked slices)
            } else {
                const bool swz = F.swz == 1 || (F.swz == 2 && range_dense(c_up, qe - qs));
                uint32_t straddle = 0;
                if (kDelta) {
                    uint32_t wb;
                    if (ubuf) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(wb) : "r"(ubuf - 4u) : "memory");
                    else wb = r_word(R, qs - 4);
                    straddle = tail_value(wb);
                }
                const uint32_t carry = kDelta ? csum - straddle + prev0 : 0u;
                RangeOut ro;
                // (plain streams: the common units -- staged, whole, before the count limit --
                // through the range-logic-free instantiation)
                const bool in_unit = !kDelta && up >= u_first && up < u_end && base + c_up < S.count;
                if (!kDelta && in_unit && swz)
                    decode_unit_ll<kDelta, true, !kDelta>(R, qs, qe, base, carry, S.count, S.out, stage, ubuf, lane, K,
                                                          ro, pol);
                else if (!kDelta && in_unit)
                    decode_unit_ll<kDelta, false, !kDelta>(R, qs, qe, base, carry, S.count, S.out, stage, ubuf, lane, K,
                                                           ro, pol);
                else if (swz)
                    decode_unit_ll<kDelta, true>(R, qs, qe, base, carry, S.count, S.out, stage, ubuf, lane, K,
                                                 ro, pol);
                else
                    decode_unit_ll<kDelta, false>(R, qs, qe, base, carry, S.count, S.out, stage, ubuf, lane, K,
                                                  ro, pol);
            }
        }
    };
    auto load_unit = [&](uint32_t u, int b) -> bool {  // TMA of unit u into buffer b (if it is staged)
        const bool full = u >= u_first && u < u_end;
        const bool st = full || u == u_part;  // (warp-uniform)
        if (st && lane == 0) {
            const uint8_t* const src = R.ab + static_cast<long long>(u) * kUnit;
            const uint32_t bytes = full ? static_cast<uint32_t>(kUnit) : part_bytes & ~15u;
            if (u == 0) tma_bulk_load(buf0 + b * kUnitBuf + 16u, src, bytes, bar0 + 8u * b);
            else tma_bulk_load(buf0 + b * kUnitBuf, src - 16, bytes + 16u, bar0 + 8u * b);
        }
        return st;
    };
    // wait for unit u's bytes in buffer b; the edge units' shared-memory fix-ups
    auto wait_unit = [&](uint32_t u, int b) {
        while (!mbar_test(bar0 + 8u * b, (phases >> b) & 1u)) {
        }
        phases ^= 1u << b;
        if (u == 0 || u == u_part) {
            const uint32_t ub = buf0 + b * kUnitBuf;
            if (u == 0 && lane < 4) asm volatile("st.shared.u32 [%0], %1;" ::"r"(ub + 4u * lane), "r"(0u) : "memory");
            if (u == u_part) {
                const uint32_t tb = part_bytes & ~15u;
                if (lane < 16) {
                    const uint32_t v = static_cast<uint32_t>(lane) < part_bytes - tb
                                           ? R.ab[static_cast<long long>(u) * kUnit + tb + lane]
                                           : 0u;
                    asm volatile("st.shared.u8 [%0], %1;" ::"r"(ub + 16u + tb + lane), "r"(v) : "memory");
                }
                for (uint32_t o = tb + 16u + 16u * lane; o < static_cast<uint32_t>(kUnit); o += 512u)
                    asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(ub + 16u + o), "r"(0u) : "memory");
            }
            __syncwarp();
        }
    };
    // totals of the staged unit u in buffer b (the zeros after a partial unit's
    // bytes count as integers -- the first may close one the stream leaves
    // unfinished -- and add nothing to the sum)
    auto staged_totals = [&](uint32_t u, int b, unsigned& c_u, uint32_t& su, uint32_t& f_u) {
        unit_totals<kDelta, kLong>(buf0 + b * kUnitBuf + 16u, kUnit / kLLSlice, lane, c_u, su, f_u);
        if (u == u_part) c_u -= static_cast<unsigned>(kUnit) - part_bytes;
    };
    // (kStatic0: the first round of units is handed out statically, unit = the warp's
    // index in the grid -- 2368 atomics on one counter took the first 4 us of every
    // launch, c2 40.1 -> 37.5 us -- and the tickets count on from there; long streams
    // keep tickets throughout: c4 measured 0.3% slower with the static round)
    const uint32_t t_off = (kMode == 0 && kStatic0) ? gridDim.x * kSegWarps : 0u;
    auto take_ticket = [&]() -> uint32_t {
        unsigned t = 0;
        if (lane == 0) {
            t = atomicAdd(ticket, 1u);
#if MVB_F_PF
            // L2 prefetch of the unit about one round of tickets ahead (whichever warp
            // takes it): its TMA load then finds the bytes in L2
            const uint32_t v = (kMode == 1 ? n_units - 1u - t : t + t_off) + (kMode == 1 ? 0u - pf_dist : pf_dist);
            if (v >= u_first && v < u_end)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(R.ab + static_cast<long long>(v) * kUnit),
                             "r"(static_cast<uint32_t>(kUnit))
                             : "memory");
#endif
        }
        return __shfl_sync(0xFFFFFFFFu, t, 0);
    };
    if constexpr (kMode == 1) {
        // totals only, last unit first: the decode pass that follows starts
        // with the units read last, still in L2
        for (;;) {
            const uint32_t t = take_ticket();
            if (t >= n_units) break;
            const uint32_t u = n_units - 1u - t;
            unsigned c_u;
            uint32_t su, f_u;
            if (load_unit(u, 0)) {
                wait_unit(u, 0);
                staged_totals(u, 0, c_u, su, f_u);
            } else {
                const long long qs = static_cast<long long>(u) * kUnit;
                fused_totals<kDelta>(S, qs, qs + kUnit, lane, c_u, su, 0u, &f_u);
            }
            fused_publish(F, 0, u, c_u, su, tag, lane, f_u);
            __syncwarp();
        }
        fused_complete(F, tag);
        return;
    }
    if constexpr (kMode == 2) {
        // decode only: every prefix is out; the next unit's bytes load while
        // this one is decoded
        uint32_t u = take_ticket();
        int b = 0;
        bool st = u < n_units && load_unit(u, b);
        while (u < n_units) {
            const uint32_t un = take_ticket();
            const bool stn = un < n_units && load_unit(un, b ^ 1);
            PrefixLoads P;
            fused_prefix_issue(F, u, lane, P);
            unsigned long long base, c_e;
            uint32_t csum, s_e;
            fused_prefix_finish(F, u, tag, lane, P, base, csum);
            const FEntry* e = F.tree[0] + u;
            fentry_get(e, tag, c_e, s_e);
            const uint32_t f_e = static_cast<uint32_t>((__ldcg(&e->s) >> 24) & 0xFFu);
            if (st) wait_unit(u, b);
            if (base < S.count) decode_unit(u, b, base, csum, static_cast<unsigned>(c_e), f_e);
            __syncwarp();  // (buffer b is refilled next iteration)
            u = un;
            st = stn;
            b ^= 1;
        }
#if MVB_BULK_OUT
        stage_wait_all(lane);
#endif
        fused_complete(F, tag);
        return;
    }
    if constexpr (kMode == 0) {
        // Pipeline per warp: take unit u, load it, total it and publish -- then
        // decode the unit taken one iteration earlier (its predecessors took their
        // tickets before it and published right after, so its prefix is out).
        // The publication must follow the ticket closely: a unit is waited for by
        // every later one.  (Measured: decoding even one slice of the previous
        // unit between the ticket and the totals, to hide the load's latency,
        // made c4 four times slower -- the delays chain from unit to unit.)
        bool have_up = false, have_first = false;
        uint32_t up = 0;  // the unit awaiting its decode (buffer bp)
        int bp = 0;
        unsigned c_up = 0;  // its totals pass: integer count, flags
        uint32_t f_up = 0;
        for (;;) {
            uint32_t u;
            if (kStatic0 && !have_first) {
                have_first = true;
                u = blockIdx.x * kSegWarps + wid;
#if MVB_F_PF
                if (lane == 0 && u + pf_dist >= u_first && u + pf_dist < u_end)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(R.ab + static_cast<long long>(u + pf_dist) * kUnit),
                                 "r"(static_cast<uint32_t>(kUnit))
                                 : "memory");
#endif
            } else {
                u = t_off + take_ticket();
            }
            MVB_FT(3);
#if MVB_F_TRACE
            if (lane == 0 && g_ftrace) {  // (the unit taken, as a pseudo-event of code 9)
                unsigned long long* row = g_ftrace + 64ull * (blockIdx.x * kSegWarps + wid);
                if (row[0] < 62) {
                    row[1 + row[0]] = (static_cast<unsigned long long>(u) << 4) | 9ull;
                    row[0] += 1;
                }
            }
#endif
            const int b = bp ^ 1;
            unsigned c_u = 0;
            uint32_t f_u = 0;
            const bool u_staged = u < n_units && load_unit(u, b);
            // unit up's prefix entries (published about an iteration ago): the loads
            // fly while unit u's bytes arrive
            PrefixLoads P;
            unsigned long long base = 0;
            uint32_t csum = 0;
            if (have_up) {
                fused_prefix_issue(F, up, lane, P);
                if (!MVB_F_LATE) fused_prefix_finish(F, up, tag, lane, P, base, csum);
                MVB_FT(6);
            }
            if (u < n_units) {
                uint32_t su;
                if (u_staged) {
                    wait_unit(u, b);
                    MVB_FT(4);
                    staged_totals(u, b, c_u, su, f_u);
                } else {
                    const long long qs = static_cast<long long>(u) * kUnit;
                    fused_totals<kDelta>(S, qs, qs + kUnit, lane, c_u, su, 0u, &f_u);
                }
                fused_publish(F, 0, u, c_u, su, tag, lane, f_u);
                MVB_FT(5);
            }
            if (have_up) {
                if (MVB_F_LATE) fused_prefix_finish(F, up, tag, lane, P, base, csum);
                decode_unit(up, bp, base, csum, c_up, f_up);
                __syncwarp();  // (buffer bp is refilled next iteration)
                MVB_FT(7);
            }
            if (u >= n_units) break;
            have_up = true;
            up = u;
            bp = b;
            c_up = c_u;
            f_up = f_u;
        }
#if MVB_BULK_OUT
        stage_wait_all(lane);
#endif
        MVB_FT(8);
    }
    fused_complete(F, tag);
}

}  // namespace mvbk
