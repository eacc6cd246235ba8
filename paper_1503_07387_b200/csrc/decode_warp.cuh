// decode_warp.cuh -- warp-autonomous, software-pipelined strict-mode decoder.
//
// Each warp of a persistent grid runs its own pipeline over 512-byte
// "warp-tiles" (tile t_i = global warp id + i * total warps), with no
// CTA-wide barrier anywhere in the steady state:
//
//   1. lane 0 prefetches t_{i+1} (512 B + 16-byte halos) into the warp's
//      shared-memory buffer with a 1-D TMA bulk copy (cp.async.bulk +
//      mbarrier) while the warp works on t_i;
//   2. the warp issues the lookback polls for t_{i-2} right away; they are
//      consumed only after t_i is decoded, so the round trip is hidden;
//   3. phase 1 (16 bytes per lane): terminator mask, integer count, warp
//      scan; the count aggregate is published; V[] (digits of p..p+4) and
//      the packed end positions EP[] go to the warp's shared memory;
//   4. phase 2: octets of 8 consecutive integers per lane (1 or 2 passes),
//      value = V[start] & bmsk(7L); delta mode scans them and publishes the
//      gap-sum aggregate;
//   5. t_{i-2}'s exclusive prefixes are resolved from the polled
//      descriptors (three-level decoupled lookback: tiles, groups of 32
//      tiles, supergroups of 32 groups; one round covers the whole in-flight
//      window), its inclusive prefixes published, and its parked values
//      written out as 16-byte-aligned streaming quads;
//   6. t_i's values (delta: in-tile inclusive prefix) are parked in the
//      warp's double-buffered VAL slot.
//
// The DecodeResult's stream positions are recovered at finalize from the
// published inclusive counts (finalize_warp), as in decode_pipelined.cuh.
//
// Replaces the reference's stream loop (/root/reference/proj/core/src/
// stream_loop.hpp:31-129) for DecodeMode::strict; semantics as in
// decode_kernel.cuh (oracle: vbyte.cpp:47-74, internal.hpp:22-37).
#pragma once

#include "decode_pipelined.cuh"

namespace mvbk {

constexpr int kWTile = 512;                 // input bytes per warp-tile
constexpr int kWInBuf = kWTile + 2 * kHalo;  // + halos
constexpr int kWV = kWTile + kHalo + 16;     // V words (local positions 0 .. 16+512, padded)
constexpr int kWEP = 4 + kWTile + 12;        // EP words: [3] = previous end, [4 + i] = end of int i
constexpr int kWVal = kWTile;                // values per parked warp-tile
constexpr int kWWarps = 8;                   // warps per CTA
constexpr int kWThreads = 32 * kWWarps;
constexpr int kL = 32;                       // lookback fan-out per level

// Per-warp shared-memory slab (bytes); every region 16-byte aligned.
constexpr int kWsIn = 0;
constexpr int kWsV = kWsIn + 2 * kWInBuf;
constexpr int kWsEP = kWsV + 4 * kWV;
constexpr int kWsVal = kWsEP + 4 * kWEP;
constexpr int kWsBar = kWsVal + 2 * 4 * kWVal;
constexpr int kWsSlab = kWsBar + 16;
constexpr int kWSmemBytes = kWWarps * kWsSlab;
static_assert(kWsV % 16 == 0 && kWsEP % 16 == 0 && kWsVal % 16 == 0 && kWsBar % 16 == 0 && kWsSlab % 16 == 0,
              "aligned slab regions");

// Three-level lookback state for one component (count or gap sum) of one
// tile: lane l holds the level-0 entry t-1-l (l < k0), the level-1 entry
// g-1-l (l < k1) and the level-2 entry s-1-l.
struct LB3 {
    unsigned long long w0, w1, w2;
    unsigned s0, s1, s2;
};

template <bool kWide>
__device__ __forceinline__ void lb3_poll(LB3& L, const unsigned long long* d0, const unsigned long long* d1,
                                         const unsigned long long* d2, long long t, long long base2,
                                         unsigned long long epoch, int lane) {
    const long long g = t >> 5, sg = g >> 5;
    const int k0 = static_cast<int>(t & 31), k1 = static_cast<int>(g & 31);
    if (lane < k0 && L.s0 == 0) {
        L.w0 = ld_relaxed(d0 + (t - 1 - lane));
        L.s0 = desc_status<kWide>(L.w0, epoch);
    }
    if (lane < k1 && L.s1 == 0) {
        L.w1 = ld_relaxed(d1 + (g - 1 - lane));
        L.s1 = desc_status<kWide>(L.w1, epoch);
    }
    if (L.s2 == 0) {
        const long long e = base2 - lane;
        if (e >= 0) {
            L.w2 = ld_relaxed(d2 + e);
            L.s2 = desc_status<kWide>(L.w2, epoch);
        } else {
            L.w2 = 0;
            L.s2 = static_cast<unsigned>(ST_INCL);
        }
    }
    (void)sg;
}

// Evaluates a polled state.  Returns true when the exclusive prefix is
// complete (written to *acc); otherwise the caller re-polls (entries that
// are needed but unpublished) or, if *advance, continues with the next 32
// supergroups (base2 -= 32) after adding them to *acc.
template <bool kWide>
__device__ __forceinline__ bool lb3_eval(const LB3& L, long long t, int lane, unsigned long long* acc,
                                         bool* advance) {
    const long long g = t >> 5;
    const int k0 = static_cast<int>(t & 31), k1 = static_cast<int>(g & 31);
    *advance = false;
    const unsigned i0 = __ballot_sync(0xFFFFFFFFu, lane < k0 && L.s0 == ST_INCL);
    const int stop0 = i0 ? __ffs(i0) - 1 : k0;
    if (__any_sync(0xFFFFFFFFu, lane < stop0 && L.s0 == 0)) return false;
    unsigned long long v = (lane < stop0 || (i0 && lane == stop0)) ? desc_value<kWide>(L.w0) : 0ull;
    bool done = i0 != 0;
    if (!done) {
        const unsigned i1 = __ballot_sync(0xFFFFFFFFu, lane < k1 && L.s1 == ST_INCL);
        const int stop1 = i1 ? __ffs(i1) - 1 : k1;
        if (__any_sync(0xFFFFFFFFu, lane < stop1 && L.s1 == 0)) return false;
        if (lane < stop1 || (i1 && lane == stop1)) v += desc_value<kWide>(L.w1);
        done = i1 != 0;
        if (!done) {
            const unsigned i2 = __ballot_sync(0xFFFFFFFFu, L.s2 == ST_INCL);
            const int stop2 = i2 ? __ffs(i2) - 1 : 32;
            if (__any_sync(0xFFFFFFFFu, lane < stop2 && L.s2 == 0)) return false;
            if (lane < stop2 || (i2 && lane == stop2)) v += desc_value<kWide>(L.w2);
            done = i2 != 0;
            *advance = !done;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    *acc += v;
    return done;
}

// Exclusive prefix of tile t for one component (blocking until resolvable).
template <bool kWide>
__device__ unsigned long long lb3_resolve(LB3& L, const unsigned long long* d0, const unsigned long long* d1,
                                          const unsigned long long* d2, long long t, unsigned long long epoch,
                                          int lane) {
    long long base2 = ((t >> 5) >> 5) - 1;
    unsigned long long acc = 0;
    unsigned backoff = 32;
    while (true) {
        bool adv;
        unsigned long long part = 0;
        if (lb3_eval<kWide>(L, t, lane, &part, &adv)) return acc + part;
        if (adv) {
            // all 32 supergroups were aggregates: keep them, look further back
            acc += part;
            base2 -= 32;
            L.s0 = ST_INCL;  // levels 0/1 are already accounted for
            L.w0 = 0;
            L.s1 = ST_INCL;
            L.w1 = 0;
            L.s2 = 0;
            // from now on levels 0 and 1 contribute nothing: mark them as empty
            // by pretending the tile and group are first in their parents
            t = (t >> 10) << 10;
        } else {
            __nanosleep(backoff);  // short cap: a sleeping poller adds its sleep to the chain
            backoff = backoff < 256 ? backoff * 2 : 256;
        }
        lb3_poll<kWide>(L, d0, d1, d2, t, base2, epoch, lane);
    }
}

// Publishes tile t's aggregate value v and rolls it up into its group and
// supergroup accumulators (last arrival publishes the parent aggregate).
template <bool kWide>
__device__ __forceinline__ void lb3_publish_agg(unsigned long long* d0, unsigned long long* d1,
                                                unsigned long long* d2, unsigned long long* a1,
                                                unsigned long long* a2, long long t, long long n_tiles,
                                                unsigned long long v, unsigned long long epoch) {
    const long long g = t >> 5, sg = g >> 5;
    const long long n_groups = (n_tiles + 31) >> 5;
    st_relaxed(d0 + t, desc_word<kWide>(t == 0 ? ST_INCL : ST_AGG, epoch, v));
    const unsigned long long old = atomicAdd(a1 + g, (1ull << 48) | v);
    const long long gsize = n_tiles - (g << 5) < 32 ? n_tiles - (g << 5) : 32;
    if (static_cast<long long>(old >> 48) + 1 == gsize) {
        const unsigned long long gt = (old + v) & (kWide ? 0xFFFFFFFFull : 0xFFFFFFFFFFFFull);
        st_relaxed(d1 + g, desc_word<kWide>(g == 0 ? ST_INCL : ST_AGG, epoch, gt));
        const unsigned long long old2 = atomicAdd(a2 + sg, (1ull << 48) | gt);
        const long long ssize = n_groups - (sg << 5) < 32 ? n_groups - (sg << 5) : 32;
        if (static_cast<long long>(old2 >> 48) + 1 == ssize)
            st_relaxed(d2 + sg, desc_word<kWide>(sg == 0 ? ST_INCL : ST_AGG, epoch, old2 + gt));
    }
}

// Publishes tile t's inclusive prefix, and its group's / supergroup's when t
// closes them.
template <bool kWide>
__device__ __forceinline__ void lb3_publish_incl(unsigned long long* d0, unsigned long long* d1,
                                                 unsigned long long* d2, long long t, long long n_tiles,
                                                 unsigned long long incl, unsigned long long epoch) {
    st_relaxed(d0 + t, desc_word<kWide>(ST_INCL, epoch, incl));
    const long long g = t >> 5;
    if ((t & 31) == 31 || t == n_tiles - 1) {
        st_relaxed(d1 + g, desc_word<kWide>(ST_INCL, epoch, incl));
        const long long n_groups = (n_tiles + 31) >> 5;
        if ((g & 31) == 31 || g == n_groups - 1) st_relaxed(d2 + (g >> 5), desc_word<kWide>(ST_INCL, epoch, incl));
    }
}

struct WParams {
    Params p;                   // stream, output, header, tile count descriptors (p.dcnt), p.dsum
    unsigned long long* g1cnt;  // level-1 (group) descriptors
    unsigned long long* g1sum;
    unsigned long long* g2cnt;  // level-2 (supergroup) descriptors
    unsigned long long* g2sum;
    unsigned long long* a1cnt;  // accumulators (zeroed by the finalizing CTA)
    unsigned long long* a1sum;
    unsigned long long* a2cnt;
    unsigned long long* a2sum;
    long long n_groups;
    long long n_super;
};

__device__ __forceinline__ long long wtile_pos0(const Params& P, long long t) { return t * kWTile - P.mis; }
__device__ __forceinline__ bool wtile_interior(const Params& P, long long t) {
    const long long p = wtile_pos0(P, t);
    return p - kHalo >= 0 && p + kWTile + kHalo <= P.len;
}

// Position just after the k-th (0-based) integer end of warp-tile t
// (computed by warp 0 of the finalizing CTA).
__device__ long long wtile_end_after(const Params& P, long long t, unsigned k, int lane) {
    const long long p0 = wtile_pos0(P, t) + 16ll * lane;
    const uint32_t e = chunk_ends(P, p0);
    const unsigned n = __popc(e);
    unsigned incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    const unsigned before = incl - n;
    long long r = 0;
    if (k >= before && k < incl) {
        uint32_t m = e;
        for (unsigned q = k - before; q > 0; --q) m &= m - 1;
        r = p0 + (__ffs(m) - 1) + 1;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xFFFFFFFFu, r, o);
    return r;
}

__device__ void finalize_warp(const WParams& W, unsigned long long epoch, int tid) {
    const Params& P = W.p;
    __threadfence();
    for (long long i = tid; i < W.n_groups; i += kWThreads) {
        W.a1cnt[i] = 0;
        W.a1sum[i] = 0;
    }
    for (long long i = tid; i < W.n_super; i += kWThreads) {
        W.a2cnt[i] = 0;
        W.a2sum[i] = 0;
    }
    if (tid >= 32) return;
    const int lane = tid;
    const long long nt = P.n_tiles;
    const unsigned long long total = tile_incl_count(P, nt - 1);
    WsHeader* h = P.hdr;
    const unsigned long long epos_inv = *reinterpret_cast<volatile unsigned long long*>(&h->err_pos_inv);
    mvb_result r;
    r.reserved = 0;
    bool done = false;
    if (epos_inv != 0ull) {
        const long long s = static_cast<long long>(~epos_inv);
        const long long ts = (s + P.mis) / kWTile;
        const long long p0 = wtile_pos0(P, ts) + 16ll * lane;
        uint32_t e = chunk_ends(P, p0);
        if (p0 >= s) e = 0;
        else if (p0 + 16 > s) e &= (1u << (s - p0)) - 1u;
        unsigned n = __popc(e);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xFFFFFFFFu, n, o);
        const unsigned long long idx = tile_incl_count(P, ts - 1) + n;
        if (idx < P.count) {
            r.status = MVB_MALFORMED;
            r.values_written = idx;
            r.bytes_consumed = static_cast<unsigned long long>(s);
            done = true;
        }
    }
    if (!done && total >= P.count) {
        long long lo = 0, hi = nt - 1;
        while (lo < hi) {
            const long long mid = (lo + hi) / 2;
            if (tile_incl_count(P, mid) >= P.count) hi = mid; else lo = mid + 1;
        }
        const unsigned k = static_cast<unsigned>(P.count - 1 - tile_incl_count(P, lo - 1));
        r.status = MVB_OK;
        r.values_written = P.count;
        r.bytes_consumed = static_cast<unsigned long long>(wtile_end_after(P, lo, k, lane));
    } else if (!done) {
        long long tl = nt - 1;
        while (tl >= 0 && tile_incl_count(P, tl) == tile_incl_count(P, tl - 1)) --tl;
        long long end = 0;
        if (tl >= 0) {
            const unsigned k = static_cast<unsigned>(tile_incl_count(P, tl) - tile_incl_count(P, tl - 1) - 1);
            end = wtile_end_after(P, tl, k, lane);
        }
        r.status = MVB_TRUNCATED;
        r.values_written = total;
        r.bytes_consumed = static_cast<unsigned long long>(end);
    }
    if (lane == 0) {
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

template <bool kDelta>
__global__ void __launch_bounds__(kWThreads, 3) vbyte_decode_warp(WParams W) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ bool s_last;
    const Params& P = W.p;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    uint8_t* const slab = smem + warp * kWsSlab;
    uint8_t* const IN0 = slab + kWsIn;
    uint32_t* const V = reinterpret_cast<uint32_t*>(slab + kWsV);
    uint32_t* const EP = reinterpret_cast<uint32_t*>(slab + kWsEP);
    uint32_t* const VAL0 = reinterpret_cast<uint32_t*>(slab + kWsVal);
    unsigned long long* const bar = reinterpret_cast<unsigned long long*>(slab + kWsBar);

    const long long nt = P.n_tiles;
    const unsigned long long epoch = P.hdr->epoch + 1;
    constexpr uint32_t kStep = (4u << 16) | 7u;
    const int lp0 = kHalo + lane * kChunk;
    const uint32_t x0 = static_cast<uint32_t>(lp0 + 1) * kStep;

    // Tiles are handed out dynamically (one ticket per warp-tile), so the
    // tiles in flight always form a compact window: every predecessor of a
    // tile was taken earlier by a warp that is making progress.  A static
    // round-robin assignment let fast warps run ahead and then stall in the
    // lookback on the slowest warp.
    long long t_next = -1;
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        t_next = static_cast<long long>(atomicAdd(&P.hdr->ticket, 1ull));
        if (t_next < nt && wtile_interior(P, t_next)) {
            mbar_expect_tx(&bar[0], kWInBuf);
            tma_load_1d(IN0, P.in + wtile_pos0(P, t_next) - kHalo, kWInBuf, &bar[0]);
        }
    }
    t_next = __shfl_sync(0xFFFFFFFFu, t_next, 0);
    __syncwarp();

    unsigned uses0 = 0, uses1 = 0;
    unsigned nt_lag0 = 0, nt_lag1 = 0;  // integer counts of t_{i-1}, t_{i-2}
    uint32_t ts_lag0 = 0, ts_lag1 = 0;  // gap sums of t_{i-1}, t_{i-2} (delta)
    long long tl0 = -1, tl1 = -1;       // tile ids of t_{i-1}, t_{i-2} (-1: none)

    for (int i = 0;; ++i) {
        const long long t = t_next < nt ? t_next : -1;  // this iteration's tile (-1: drain)
        const bool have_cur = t >= 0;
        if (!have_cur && tl0 < 0 && tl1 < 0) break;
        const int cb = i & 1;
        uint8_t* const inb = IN0 + cb * kWInBuf;
        uint32_t* const vals = VAL0 + cb * kWVal;  // t_i's slot == t_{i-2}'s slot

        // ---- take and prefetch the next tile ----
        if (have_cur) {
            if (lane == 0) {
                t_next = static_cast<long long>(atomicAdd(&P.hdr->ticket, 1ull));
                if (t_next < nt && wtile_interior(P, t_next)) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect_tx(&bar[cb ^ 1], kWInBuf);
                    tma_load_1d(IN0 + (cb ^ 1) * kWInBuf, P.in + wtile_pos0(P, t_next) - kHalo, kWInBuf,
                                &bar[cb ^ 1]);
                }
            }
            t_next = __shfl_sync(0xFFFFFFFFu, t_next, 0);
        }

        // ---- issue the lookback polls for t_{i-2} (consumed after phase 2) ----
        const long long tp = tl1;
        const bool have_prev = tp > 0;
        LB3 lc = {0, 0, 0, 0, 0, 0}, ls = {0, 0, 0, 0, 0, 0};
        if (have_prev) {
            const long long base2 = ((tp >> 5) >> 5) - 1;
            lb3_poll<false>(lc, P.dcnt, W.g1cnt, W.g2cnt, tp, base2, epoch, lane);
            if (kDelta) lb3_poll<true>(ls, P.dsum, W.g1sum, W.g2sum, tp, base2, epoch, lane);
        }

        uint32_t val[kPasses][8];
        unsigned n_tile = 0;
        uint32_t tile_sum = 0;
        if (have_cur) {
            // ---- input ----
            const bool interior = wtile_interior(P, t);
            if (interior) {
                const unsigned u = cb ? uses1 : uses0;
                while (!mbar_try_wait(&bar[cb], u & 1)) {
                }
                if (cb) ++uses1; else ++uses0;
            } else {
                const long long base = wtile_pos0(P, t) - kHalo;
                for (int k = lane; k < kWInBuf; k += 32) inb[k] = static_cast<uint8_t>(byte_at(P, base + k));
                __syncwarp();
            }
            // ---- phase 1 ----
            const uint4 q = *reinterpret_cast<const uint4*>(inb + lp0);
            const uint2 pv = *reinterpret_cast<const uint2*>(inb + lp0 - 8);
            const uint32_t w0 = q.x, w1 = q.y, w2 = q.z, w3 = q.w, wp2 = pv.x, wp3 = pv.y;
            const uint32_t wn = *reinterpret_cast<const uint32_t*>(inb + lp0 + kChunk);
            const uint32_t T16 = hibits16(~w0, ~w1, ~w2, ~w3);
            const uint32_t Tx = (hibits4(~wp2) | (hibits4(~wp3) << 4)) | (T16 << 8) | (hibits4(~wn) << 24);
            const uint32_t Cx = ~Tx & 0x0FFFFFFFu;
            uint32_t inr16 = 0xFFFFu;
            if (!interior) {
                const long long p0 = wtile_pos0(P, t) + static_cast<long long>(lane) * kChunk;
                const long long lo = p0 < 0 ? -p0 : 0;
                const long long hi = P.len - p0 < 16 ? P.len - p0 : 16;
                inr16 = (hi <= lo) ? 0u : ((0xFFFFu >> (16 - (hi - lo))) << lo) & 0xFFFFu;
            }
            const uint32_t ends16 = T16 & inr16;
            const uint32_t five = (Tx >> 3) & (Cx >> 4) & (Cx >> 5) & (Cx >> 6) & (Cx >> 7) & inr16;
            if (five) {
                const uint32_t g0 = w0 | (w0 << 1) | (w0 << 2) | (w0 << 3);
                const uint32_t g1 = w1 | (w1 << 1) | (w1 << 2) | (w1 << 3);
                const uint32_t g2 = w2 | (w2 << 1) | (w2 << 2) | (w2 << 3);
                const uint32_t g3 = w3 | (w3 << 1) | (w3 << 2) | (w3 << 3);
                const uint32_t bad16 = five & hibits16(g0, g1, g2, g3);
                if (bad16) {  // start of a malformed integer (index recovered at finalize)
                    const long long s = wtile_pos0(P, t) + static_cast<long long>(lane) * kChunk + (__ffs(bad16) - 1) - 4;
                    atomicMax(&P.hdr->err_pos_inv, ~static_cast<unsigned long long>(s));
                }
            }
            const unsigned n_own = __popc(ends16);
            unsigned incl = n_own;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= o) incl += y;
            }
            n_tile = __shfl_sync(0xFFFFFFFFu, incl, 31);
            const unsigned tbase = incl - n_own;
            if (lane == 0)
                lb3_publish_agg<false>(P.dcnt, W.g1cnt, W.g2cnt, W.a1cnt, W.a2cnt, t, nt, n_tile, epoch);
            // ---- V and packed end positions ----
            const uint32_t d0 = digits4(w0), d1 = digits4(w1), d2 = digits4(w2), d3 = digits4(w3), dn = digits4(wn);
            uint4* vq = reinterpret_cast<uint4*>(V + lp0);
            vq[0] = vquad(d0, d1);
            vq[1] = vquad(d1, d2);
            vq[2] = vquad(d2, d3);
            vq[3] = vquad(d3, dn);
            if (lane == 0) {  // halo positions -8..-1 (local 8..15)
                const uint32_t dp2 = digits4(wp2), dp3 = digits4(wp3);
                uint4* hq = reinterpret_cast<uint4*>(V + 8);
                hq[0] = vquad(dp2, dp3);
                hq[1] = vquad(dp3, d0);
                const uint32_t tp8 = Tx & 0xFFu;  // positions -8..-1
                const unsigned prev_lp = (t == 0) ? static_cast<unsigned>(kHalo - 1 + P.mis)
                                         : tp8    ? static_cast<unsigned>(8 + 31 - __clz(tp8))
                                                  : 7u;
                EP[3] = (prev_lp + 1) * kStep;
            }
            {
                uint32_t* ep = EP + 4 + tbase;
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
            }
            __syncwarp();
            // ---- phase 2: octets u = lane + 32p ----
            uint32_t carry_in = 0;  // delta: running sum of earlier passes
#pragma unroll
            for (int p = 0; p < kPasses; ++p) {
#pragma unroll
                for (int k = 0; k < 8; ++k) val[p][k] = 0;
                if (256 * p >= static_cast<int>(n_tile)) continue;  // warp-uniform
                const unsigned u = lane + 32 * p;
                if (8 * u < n_tile) {
                    const uint4 qa = *reinterpret_cast<const uint4*>(EP + 4 + 8 * u);
                    const uint4 qb = *reinterpret_cast<const uint4*>(EP + 8 + 8 * u);
                    const uint32_t xs[9] = {EP[3 + 8 * u], qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
#pragma unroll
                    for (int k = 0; k < 8; ++k) val[p][k] = lds_at(V, xs[k] >> 16) & bmsk((xs[k + 1] - xs[k]) & 0xFFFFu);
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
                    const uint32_t ex = carry_in + x - val[p][7];
#pragma unroll
                    for (int k = 0; k < 8; ++k) val[p][k] += ex;
                    carry_in += __shfl_sync(0xFFFFFFFFu, x, 31);
                }
            }
            tile_sum = carry_in;
            if (kDelta && lane == 0)
                lb3_publish_agg<true>(P.dsum, W.g1sum, W.g2sum, W.a1sum, W.a2sum, t, nt,
                                      t == 0 ? static_cast<uint32_t>(prev_of(P) + tile_sum) : tile_sum, epoch);
        }

        // ---- resolve and store t_{i-2} ----
        if (tl1 >= 0) {
            unsigned long long cnt_prefix = 0;
            uint32_t carry = prev_of(P);
            if (have_prev) {
                cnt_prefix = lb3_resolve<false>(lc, P.dcnt, W.g1cnt, W.g2cnt, tp, epoch, lane);
                if (kDelta) carry = static_cast<uint32_t>(lb3_resolve<true>(ls, P.dsum, W.g1sum, W.g2sum, tp, epoch, lane));
                if (lane == 0) {
                    lb3_publish_incl<false>(P.dcnt, W.g1cnt, W.g2cnt, tp, nt, cnt_prefix + nt_lag1, epoch);
                    if (kDelta)
                        lb3_publish_incl<true>(P.dsum, W.g1sum, W.g2sum, tp, nt,
                                               static_cast<uint32_t>(carry + ts_lag1), epoch);
                }
            }
            if (!kDelta) carry = 0;
            const unsigned long long room = P.count > cnt_prefix ? P.count - cnt_prefix : 0ull;
            const unsigned lim = room < nt_lag1 ? static_cast<unsigned>(room) : nt_lag1;
            const unsigned a = static_cast<unsigned>(((reinterpret_cast<uintptr_t>(P.out) >> 2) + cnt_prefix) & 3u);
            uint32_t* const qbase = P.out + cnt_prefix - a;
            const unsigned nq = lim ? (lim + a + 3) >> 2 : 0u;
            for (unsigned qi = lane; qi < nq; qi += 32) {
                const int i0 = static_cast<int>(4 * qi) - static_cast<int>(a);
                if (i0 >= 0 && static_cast<unsigned>(i0) + 4 <= lim) {
                    uint32_t v0, v1, v2, v3;
                    if (a == 0) {
                        const uint4 x = *reinterpret_cast<const uint4*>(vals + i0);
                        v0 = x.x; v1 = x.y; v2 = x.z; v3 = x.w;
                    } else if (a == 2) {
                        const uint2 x = *reinterpret_cast<const uint2*>(vals + i0);
                        const uint2 y = *reinterpret_cast<const uint2*>(vals + i0 + 2);
                        v0 = x.x; v1 = x.y; v2 = y.x; v3 = y.y;
                    } else {
                        const uint2 x = *reinterpret_cast<const uint2*>(vals + i0 + 1);
                        v0 = vals[i0]; v1 = x.x; v2 = x.y; v3 = vals[i0 + 3];
                    }
                    stg_stream16(qbase + 4 * qi, v0 + carry, v1 + carry, v2 + carry, v3 + carry);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int ii = i0 + k;
                        if (ii >= 0 && static_cast<unsigned>(ii) < lim) stg_stream4(qbase + 4 * qi + k, vals[ii] + carry);
                    }
                }
            }
            __syncwarp();
        }
        nt_lag1 = nt_lag0;
        ts_lag1 = ts_lag0;
        tl1 = tl0;
        tl0 = t;
        if (!have_cur) continue;
        nt_lag0 = n_tile;
        ts_lag0 = tile_sum;

        // ---- park t_i's values ----
#pragma unroll
        for (int p = 0; p < kPasses; ++p) {
            if (256 * p >= static_cast<int>(n_tile)) continue;
            const unsigned u = lane + 32 * p;
            uint4* dst = reinterpret_cast<uint4*>(vals + 8 * u);
            dst[0] = make_uint4(val[p][0], val[p][1], val[p][2], val[p][3]);
            dst[1] = make_uint4(val[p][4], val[p][5], val[p][6], val[p][7]);
        }
        __syncwarp();
    }

    // ---- completion; the last CTA produces the DecodeResult ----
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        s_last = atomicAdd(&P.hdr->done, 1ull) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    finalize_warp(W, epoch, tid);
}

}  // namespace mvbk
