// decode_v3.cuh -- warp-sliced, barrier-free strict-mode decoder (kernel choice 3).
//
// Status: correct (every strict-mode parity test runs it) but, as measured on
// B200, only faster than the CTA-pipelined default on all-1-byte streams
// (c5_all1 214 vs 253 us); on c2/c1/all5 it is 7-30% slower -- the lookback
// latency chain (scripts/analyze_trace3.py) and per-lane phase-2 overheads
// dominate.  Kept as the experimental variant and for its timeline trace.
//
// Same tile algorithm and lookback as vbyte_decode_pipelined
// (decode_pipelined.cuh), re-partitioned so that the eight worker warps of a
// CTA never wait for one another:
//
//   * a 4 KiB tile is cut into eight 512-byte slices, one per worker warp;
//     each warp decodes its slice end to end -- terminator scan, V (digit
//     windows), EP (integer ends), phase 2 and the final stores -- in its own
//     shared-memory regions, so phase 2 is balanced by construction (equal
//     bytes per warp) and needs no CTA-wide scatter barrier;
//   * the only CTA-level coupling is a producer/consumer pair of named
//     barriers with the lookback warp: workers `bar.arrive` when a tile's
//     per-warp counts and gap sums are in shared memory; the lookback warp
//     `bar.sync`s, takes a tile ticket three iterations ahead, prefetches the
//     tile two iterations ahead by TMA, publishes the tile's aggregates,
//     resolves its output index and carry (decoupled lookback) and
//     `bar.arrive`s; workers `bar.sync` on that only when they store the
//     tile, two iterations later -- so the lookback's global round trips hide
//     behind a whole iteration of decoding;
//   * tiles are handed out by a ticket counter in stream order, so a lookback
//     only waits on tiles started before its own;
//   * values stay parked per warp (double-buffered) until their tile's prefix
//     is known, then each warp streams its own segment out with aligned
//     16-byte stores.
//
// Shared-memory layouts are swizzled for conflict-free wavefronts
// (scripts/smem_model.py).  Semantics as in decode_kernel.cuh (oracle:
// vbyte.cpp:47-74, internal.hpp:22-37); replaces stream_loop.hpp:31-129 for
// DecodeMode::strict.
#pragma once

#include "decode_pipelined.cuh"
#include "decode_warp.cuh"

namespace mvbk {

constexpr int kV3Workers = 8;
constexpr int kV3WorkerThreads = 32 * kV3Workers;
constexpr int kV3Threads = kV3WorkerThreads + 32;
constexpr int kV3LBWarp = kV3Workers;
constexpr int kVW = 528;    // V words per warp: 8 halo positions + 512 + pad (64-byte multiple)
constexpr int kEPH = 584;   // EP halfwords per warp: [3] previous end, [4 + k] end of int k, 64 padding
constexpr int kValW = 544;  // parked values per warp: 32 lanes x K' <= 17 slots
// Named barriers (0 is __syncthreads).  Producer/consumer pairs alternate
// between two ids by tile parity, so one side running a phase ahead can never
// be counted into the other side's current phase.
constexpr unsigned kBarAgg0 = 1;  // +j&1: workers arrive, lookback warp syncs: tile t_j's per-warp totals are out
constexpr unsigned kBarPre0 = 3;  // +j&1: lookback warp arrives, workers sync: tile t_j's prefix is resolved
constexpr unsigned kBarFill = 5;  // workers only: stream-edge tile filled by hand

constexpr int kS3In = 0;
constexpr int kS3V = kS3In + 2 * kInBuf;
constexpr int kS3EP = kS3V + 4 * kV3Workers * kVW;
constexpr int kS3Val = kS3EP + 2 * kV3Workers * kEPH;
constexpr int kS3Bytes = kS3Val + 2 * 4 * kV3Workers * kValW;
static_assert(kS3V % 64 == 0 && (4 * kVW) % 64 == 0 && kS3EP % 16 == 0 && kS3Val % 16 == 0 && (2 * kEPH) % 16 == 0 &&
                  (4 * kValW) % 16 == 0,
              "alignment");

__device__ __forceinline__ void nb_sync(unsigned id, unsigned n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nb_arrive(unsigned id, unsigned n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Aggregate publication of tile t by one warp, lanes 0 (count, 40-bit
// descriptors) and 1 (gap sum, 32-bit) in lockstep: tile descriptor, group
// accumulator, and -- for the last arrival -- group descriptor and supergroup
// accumulator/descriptor (lb3_publish_agg, decode_warp.cuh, for both
// components at once: each level costs one atomic round trip, not two).
__device__ __forceinline__ void publish_agg_pair(const WParams& W, long long t, unsigned long long n_tile,
                                                 unsigned long long t_sum, unsigned long long epoch, int lane,
                                                 int ncomp) {
    if (lane >= ncomp) return;
    const Params& P = W.p;
    const bool wide = lane == 1;
    unsigned long long* const d0 = wide ? P.dsum : P.dcnt;
    unsigned long long* const d1 = wide ? W.g1sum : W.g1cnt;
    unsigned long long* const d2 = wide ? W.g2sum : W.g2cnt;
    unsigned long long* const a1 = wide ? W.a1sum : W.a1cnt;
    unsigned long long* const a2 = wide ? W.a2sum : W.a2cnt;
    const unsigned long long mask = wide ? 0xFFFFFFFFull : 0xFFFFFFFFFFFFull;
    const unsigned long long v = wide ? t_sum : n_tile;
#define MVB_DW(st, val) (wide ? desc_word<true>((st), epoch, (val)) : desc_word<false>((st), epoch, (val)))
    const long long n_tiles = P.n_tiles;
    const long long g = t >> 5, sg = g >> 5;
    st_relaxed(d0 + t, MVB_DW(t == 0 ? ST_INCL : ST_AGG, v));
    const unsigned long long old = atomicAdd(a1 + g, (1ull << 48) | v);
    const long long gsize = n_tiles - (g << 5) < 32 ? n_tiles - (g << 5) : 32;
    if (static_cast<long long>(old >> 48) + 1 == gsize) {
        const unsigned long long gt = (old + v) & mask;
        st_relaxed(d1 + g, MVB_DW(g == 0 ? ST_INCL : ST_AGG, gt));
        const unsigned long long old2 = atomicAdd(a2 + sg, (1ull << 48) | gt);
        const long long ssize = W.n_groups - (sg << 5) < 32 ? W.n_groups - (sg << 5) : 32;
        if (static_cast<long long>(old2 >> 48) + 1 == ssize)
            st_relaxed(d2 + sg, MVB_DW(sg == 0 ? ST_INCL : ST_AGG, (old2 + gt) & mask));
    }
#undef MVB_DW
}

// Optional per-tile timeline (profiling only, scripts/trace_tiles.py):
// [0] ticket  [1] phase 1 start  [2] last warp done  [3] aggregates out
// [4] lookback start  [5] prefix resolved  [6] stores start  [7] smid<<32|block
#define MVB_T3(t, k)                                                                            \
    do {                                                                                        \
        if (P.trace) P.trace[static_cast<unsigned long long>(t) * 8 + (k)] = gtimer();          \
    } while (0)

template <bool kDelta>
__global__ void __launch_bounds__(kV3Threads, 3) vbyte_decode_v3(WParams W) {
    const Params& P = W.p;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t (*IN)[kInBuf] = reinterpret_cast<uint8_t (*)[kInBuf]>(smem + kS3In);
    __shared__ __align__(8) unsigned long long bar[2];
    __shared__ unsigned s_wcnt[4][kV3Workers];
    __shared__ uint32_t s_wsum[4][kV3Workers];
    __shared__ unsigned long long s_wbase[4][kV3Workers];  // output index of each warp's first int
    __shared__ uint32_t s_wcarry[4][kV3Workers];           // delta carry into each warp's first int
    __shared__ long long s_tile[4];  // tile of iteration k at [k & 3] (dynamic tickets)
    __shared__ int s_my;             // number of tiles this CTA processes, once known
    __shared__ unsigned s_arr[4];    // worker warps done with the tile of iteration k
    __shared__ int s_tseq[4];        // iteration whose ticket s_tile[k & 3] holds (written last)
    __shared__ bool s_last;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const unsigned long long epoch = P.hdr->epoch + 1;  // constant during a launch
    constexpr int kUnknown = 0x7FFFFFF0;

    // Tiles are handed out in stream order by a ticket counter, two
    // iterations ahead of their decode: a CTA that runs slow simply takes
    // fewer tiles, so a lookback only ever waits on tiles that were started
    // before its own (static strides made every lookback wait for the
    // slowest CTA of the grid).
    if (tid == kV3WorkerThreads) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        int my = kUnknown;
        for (int k = 0; k < 2; ++k) {
            const long long t = static_cast<long long>(atomicAdd(&P.hdr->ticket, 1ull));
            if (t >= static_cast<long long>(P.n_tiles)) {
                my = k;
                break;
            }
            s_tile[k] = t;
            MVB_T3(t, 0);
            if (tile_interior(P, t)) {
                mbar_expect_tx(&bar[k], kInBuf);
                tma_load_1d(IN[k], P.in + tile_pos0(P, t) - kHalo, kInBuf, &bar[k]);
            }
        }
        s_my = my;
    }
    if (tid < 4) {
        s_arr[tid] = 0;
        s_tseq[tid] = tid < 2 ? tid : -1;
    }
    __syncthreads();

    if (warp == kV3LBWarp) {
        // ------------------------------------------------ lookback warp
        // iteration j: wait for the workers to finish t_j, take the ticket
        // of iteration j+2 and prefetch it into IN[j & 1] (free: the workers
        // are past t_j's phase 1), publish nothing (the last worker warp did),
        // and resolve t_j's prefix.  The workers store t_j in iteration j+2,
        // so the lookback has a whole worker iteration to complete.
        int my = s_my;
        for (int j = 0; j < my; ++j) {
            const long long t = s_tile[j & 3];
            nb_sync(kBarAgg0 + (j & 1), kV3Threads);
            if (j + 2 < my) {
                long long tn = 0;
                if (lane == 0) {
                    tn = static_cast<long long>(atomicAdd(&P.hdr->ticket, 1ull));
                    if (tn >= static_cast<long long>(P.n_tiles)) {
                        s_my = j + 2;
                    } else {
                        s_tile[(j + 2) & 3] = tn;
                        MVB_T3(tn, 0);
                        if (tile_interior(P, tn)) {
                            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                            mbar_expect_tx(&bar[j & 1], kInBuf);
                            tma_load_1d(IN[j & 1], P.in + tile_pos0(P, tn) - kHalo, kInBuf, &bar[j & 1]);
                        }
                    }
                    __threadfence_block();
                    *static_cast<volatile int*>(&s_tseq[(j + 2) & 3]) = j + 2;  // publish the slot
                }
                tn = __shfl_sync(0xFFFFFFFFu, tn, 0);
                if (tn >= static_cast<long long>(P.n_tiles)) my = j + 2;
            }
            const unsigned c = lane < kV3Workers ? s_wcnt[j & 3][lane] : 0u;
            const uint32_t sm = lane < kV3Workers ? s_wsum[j & 3][lane] : 0u;
            const unsigned n_tile = __reduce_add_sync(0xFFFFFFFFu, c);
            const uint32_t t_sum = __reduce_add_sync(0xFFFFFFFFu, sm);
            // (t_j's tile and group aggregates went out from its last worker warp)
            unsigned long long cp = 0;
            uint32_t cs = prev_of(P);
            if (lane == 0) MVB_T3(t, 4);
            if (t > 0) {
                LB3 lc = {0, 0, 0, 0, 0, 0}, ls = {0, 0, 0, 0, 0, 0};
                const long long base2 = ((t >> 5) >> 5) - 1;
                lb3_poll<false>(lc, P.dcnt, W.g1cnt, W.g2cnt, t, base2, epoch, lane);
                if (kDelta) lb3_poll<true>(ls, P.dsum, W.g1sum, W.g2sum, t, base2, epoch, lane);
                cp = lb3_resolve<false>(lc, P.dcnt, W.g1cnt, W.g2cnt, t, epoch, lane);
                if (kDelta) cs = static_cast<uint32_t>(lb3_resolve<true>(ls, P.dsum, W.g1sum, W.g2sum, t, epoch, lane));
                if (lane == 0) lb3_publish_incl<false>(P.dcnt, W.g1cnt, W.g2cnt, t, P.n_tiles, cp + n_tile, epoch);
                if (kDelta && lane == 1)
                    lb3_publish_incl<true>(P.dsum, W.g1sum, W.g2sum, t, P.n_tiles, static_cast<uint32_t>(cs + t_sum),
                                           epoch);
            }
            {  // per-warp output bases and carries of t_j (lanes 0..7)
                unsigned ec = c;
                uint32_t es = sm;
#pragma unroll
                for (int o = 1; o < kV3Workers; o <<= 1) {
                    const unsigned yc = __shfl_up_sync(0xFFFFFFFFu, ec, o);
                    const uint32_t ys = __shfl_up_sync(0xFFFFFFFFu, es, o);
                    if (lane >= o) {
                        ec += yc;
                        es += ys;
                    }
                }
                if (lane < kV3Workers) {
                    s_wbase[j & 3][lane] = cp + (ec - c);
                    s_wcarry[j & 3][lane] = cs + (es - sm);
                }
                if (lane == 0) MVB_T3(t, 5);
            }
            nb_arrive(kBarPre0 + (j & 1), kV3Threads);
        }
    } else {
        // ------------------------------------------------ worker warps
        char* const vbase = reinterpret_cast<char*>(smem + kS3V) + warp * (4 * kVW);
        uint16_t* const eph = reinterpret_cast<uint16_t*>(smem + kS3EP) + warp * kEPH;
        const int lp0 = kHalo + tid * kChunk;  // tile-local byte coordinate of this lane's chunk
        const uint32_t r0 = 8u + 16u * static_cast<uint32_t>(lane);  // warp-local V index of the chunk
        unsigned uses0 = 0, uses1 = 0;
        long long t_cur = -1, t_lag1 = -1, t_lag2 = -1;

        for (int i = 0;; ++i) {
            // iteration i's ticket (or the end of this CTA's tiles) is written
            // by lookback iteration i-2, which may still be under way
            if (i >= 2 && i < *static_cast<volatile int*>(&s_my)) {
                while (*static_cast<volatile int*>(&s_tseq[i & 3]) != i && i < *static_cast<volatile int*>(&s_my)) {
                }
                __threadfence_block();
            }
            const int my_tiles = *static_cast<volatile int*>(&s_my);
            if (i >= my_tiles + 2) break;
            const bool have_cur = i < my_tiles;
            const long long t = have_cur ? s_tile[i & 3] : -1;
            t_lag2 = t_lag1;  // tile of iteration i-2 (tracing only)
            t_lag1 = t_cur;
            t_cur = t;
            const int cb = i & 1;
            uint32_t* const valw = reinterpret_cast<uint32_t*>(smem + kS3Val) + (cb * kV3Workers + warp) * kValW;
            unsigned n_w = 0;

            if (have_cur) {
                // ---- phase 1: terminators, counts, V and EP of this warp's slice ----
                const uint8_t* buf = IN[cb];
                const bool interior = tile_interior(P, t);
                if (interior) {
                    const unsigned u = cb ? uses1 : uses0;
                    while (!mbar_try_wait(&bar[cb], u & 1)) {
                    }
                    if (cb) ++uses1; else ++uses0;
                } else {
                    // stream start / end: fill with padding (0x00 before, 0x80 after)
                    uint8_t* wbuf = IN[cb];
                    const long long base = tile_pos0(P, t) - kHalo;
                    for (int k = tid; k < kInBuf; k += kV3WorkerThreads)
                        wbuf[k] = static_cast<uint8_t>(byte_at(P, base + k));
                    nb_sync(kBarFill, kV3WorkerThreads);
                }
                if (tid == 0) MVB_T3(t, 1);
                const uint4 q = *reinterpret_cast<const uint4*>(buf + lp0);
                const uint32_t w0 = q.x, w1 = q.y, w2 = q.z, w3 = q.w;
                uint32_t wp2 = __shfl_up_sync(0xFFFFFFFFu, w2, 1);
                uint32_t wp3 = __shfl_up_sync(0xFFFFFFFFu, w3, 1);
                uint32_t wn = __shfl_down_sync(0xFFFFFFFFu, w0, 1);
                if (lane == 0) {
                    const uint2 pv = *reinterpret_cast<const uint2*>(buf + lp0 - 8);
                    wp2 = pv.x;
                    wp3 = pv.y;
                }
                if (lane == 31) wn = *reinterpret_cast<const uint32_t*>(buf + lp0 + kChunk);

                const uint32_t T16 = hibits16(~w0, ~w1, ~w2, ~w3);
                const uint32_t Tx = (hibits4(~wp2) | (hibits4(~wp3) << 4)) | (T16 << 8) | (hibits4(~wn) << 24);
                const uint32_t Cx = ~Tx & 0x0FFFFFFFu;
                uint32_t inr16 = 0xFFFFu;
                if (!interior) {
                    const long long p0 = tile_pos0(P, t) + static_cast<long long>(tid) * kChunk;
                    const long long lo = p0 < 0 ? -p0 : 0;
                    const long long hi = P.len - p0 < 16 ? P.len - p0 : 16;
                    inr16 = (hi <= lo) ? 0u : ((0xFFFFu >> (16 - (hi - lo))) << lo) & 0xFFFFu;
                }
                const uint32_t ends16 = T16 & inr16;
                // strict: a fifth byte >= 0x10 (4 continuation bytes after an integer end)
                if (Cx & (Cx >> 1) & (Cx >> 2) & (Cx >> 3)) {
                    const uint32_t five = (Tx >> 3) & (Cx >> 4) & (Cx >> 5) & (Cx >> 6) & (Cx >> 7) & inr16;
                    if (five) {
                        const uint32_t g0 = w0 | (w0 << 1) | (w0 << 2) | (w0 << 3);
                        const uint32_t g1 = w1 | (w1 << 1) | (w1 << 2) | (w1 << 3);
                        const uint32_t g2 = w2 | (w2 << 1) | (w2 << 2) | (w2 << 3);
                        const uint32_t g3 = w3 | (w3 << 1) | (w3 << 2) | (w3 << 3);
                        const uint32_t bad16 = five & hibits16(g0, g1, g2, g3);
                        if (bad16) {  // start of a malformed integer: s = p - 4 (index recovered at finalize)
                            const long long s =
                                tile_pos0(P, t) + static_cast<long long>(tid) * kChunk + (__ffs(bad16) - 1) - 4;
                            atomicMax(&P.hdr->err_pos_inv, ~static_cast<unsigned long long>(s));
                        }
                    }
                }
                const uint32_t n_own = __popc(ends16);
                uint32_t incl = n_own;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                    if (lane >= o) incl += y;
                }
                n_w = __shfl_sync(0xFFFFFFFFu, incl, 31);
                const uint32_t wexcl = incl - n_own;

                // V: digit window of every byte position of the slice (+ 8 halo positions)
                const uint32_t d0 = digits4(w0), d1 = digits4(w1), d2 = digits4(w2), d3 = digits4(w3),
                               dn = digits4(wn);
                const uint32_t vo = 4u * r0;
                *reinterpret_cast<uint4*>(vbase + v_swz(vo)) = vquad(d0, d1);
                *reinterpret_cast<uint4*>(vbase + v_swz(vo + 16)) = vquad(d1, d2);
                *reinterpret_cast<uint4*>(vbase + v_swz(vo + 32)) = vquad(d2, d3);
                *reinterpret_cast<uint4*>(vbase + v_swz(vo + 48)) = vquad(d3, dn);
                if (lane == 0) {  // halo positions -8..-1 of the slice
                    const uint32_t dp2 = digits4(wp2), dp3 = digits4(wp3);
                    *reinterpret_cast<uint4*>(vbase + v_swz(0)) = vquad(dp2, dp3);
                    *reinterpret_cast<uint4*>(vbase + v_swz(16)) = vquad(dp3, d0);
                }
                // EP: V indices of the slice's integer ends, in order (16-bit)
                uint16_t* ep = eph + 4 + wexcl;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if ((ends16 >> j) & 1u) {
                        *ep = static_cast<uint16_t>(r0 + j);
                        ++ep;
                    }
                }
                {  // 64 zero-width padding entries after the last end (phase 2 reads up to 32*K')
                    const unsigned hasb = __ballot_sync(0xFFFFFFFFu, n_own != 0);
                    const uint32_t rl = __shfl_sync(0xFFFFFFFFu, r0 + (31 - __clz(ends16 | 1u)), hasb ? 31 - __clz(hasb) : 0);
                    eph[4 + n_w + lane] = static_cast<uint16_t>(rl);
                    eph[4 + n_w + 32 + lane] = static_cast<uint16_t>(rl);
                }
                if (lane == 0) {
                    const uint32_t tp8 = Tx & 0xFFu;  // slice positions -8..-1 (V index 0..7)
                    const int prev_r = (t == 0 && warp == 0) ? static_cast<int>(7 + P.mis)
                                       : tp8              ? 31 - __clz(tp8)
                                                          : -1;
                    eph[3] = static_cast<uint16_t>(prev_r);  // -1 -> 0xFFFF: start index 0 after +1 (mod 2^16)
                }
                __syncwarp();
            }

            if (i >= 2) {
                nb_sync(kBarPre0 + (i & 1), kV3Threads);  // t_{i-2}'s prefix (lookback iteration i-2)
                if (tid == 0) MVB_T3(t_lag2, 6);
                // ---- store this warp's segment of t_{i-2} (parked in valw: (i-2) & 1 == cb) ----
                const int ps = (i - 2) & 3;
                const unsigned n = s_wcnt[ps][warp];
                const unsigned long long base = s_wbase[ps][warp];
                const uint32_t carry = kDelta ? s_wcarry[ps][warp] : 0u;
                const unsigned lim = base + n <= P.count ? n : (base < P.count ? static_cast<unsigned>(P.count - base) : 0u);
                const unsigned a = static_cast<unsigned>(((reinterpret_cast<uintptr_t>(P.out) >> 2) + base) & 3u);
                const unsigned h = (4u - a) & 3u;
                const unsigned hh = h < lim ? h : lim;
                const unsigned nbody = (lim - hh) >> 2;
                const unsigned tail0 = hh + 4 * nbody;
                uint32_t* const o = P.out + base;
                if (static_cast<unsigned>(lane) < hh) {
                    stg_stream4(o + lane, valw[lane] + carry);
                } else if (lane >= 4 && static_cast<unsigned>(lane - 4) < lim - tail0) {
                    stg_stream4(o + tail0 + lane - 4, valw[tail0 + lane - 4] + carry);
                }
                const uint4* const vq = reinterpret_cast<const uint4*>(valw);
                uint32_t* const ob = o + hh;
#define MVB_BODY3(H)                                                                                  \
    for (unsigned m = lane; m < nbody; m += 32) {                                                     \
        const uint4 x = vq[m];                                                                        \
        uint32_t e0, e1, e2, e3;                                                                      \
        if (H == 0) {                                                                                 \
            e0 = x.x; e1 = x.y; e2 = x.z; e3 = x.w;                                                   \
        } else {                                                                                      \
            const uint4 y = vq[m + 1];                                                                \
            if (H == 1) { e0 = x.y; e1 = x.z; e2 = x.w; e3 = y.x; }                                   \
            else if (H == 2) { e0 = x.z; e1 = x.w; e2 = y.x; e3 = y.y; }                              \
            else { e0 = x.w; e1 = y.x; e2 = y.y; e3 = y.z; }                                          \
        }                                                                                             \
        stg_stream16(ob + 4 * m, e0 + carry, e1 + carry, e2 + carry, e3 + carry);                    \
    }
                switch (h) {  // h < lim implies hh == h; otherwise nbody == 0
                    case 0: MVB_BODY3(0) break;
                    case 1: MVB_BODY3(1) break;
                    case 2: MVB_BODY3(2) break;
                    default: MVB_BODY3(3) break;
                }
#undef MVB_BODY3
                __syncwarp();  // valw is reused below
            }

            if (have_cur) {
                // ---- phase 2: values of the slice's integers, K' consecutive per lane ----
                // K' = ceil(n_w / 32) made odd, so the lane-strided EP reads and
                // VAL writes are bank-conflict-free; slots past n_w read the
                // zero-width padding and produce 0.
                uint32_t run = 0;  // delta: gap sum of the slice
                if (n_w) {
                    const unsigned Kp = ((n_w + 31) >> 5) | 1u;
                    const uint16_t* const e = eph + 3 + Kp * lane;
                    uint32_t rp = e[0];
                    uint32_t val[17];
                    uint32_t acc = 0;
#pragma unroll
                    for (int k = 0; k < 17; ++k) {
                        if (k < static_cast<int>(Kp)) {
                            const uint32_t r = e[1 + k];
                            const uint32_t v = *reinterpret_cast<const uint32_t*>(vbase + v_swz(4u * ((rp + 1u) & 0xFFFFu))) &
                                               bmsk(7u * (r - rp));
                            acc += v;
                            val[k] = kDelta ? acc : v;
                            rp = r;
                        }
                    }
                    uint32_t ex = 0;
                    if (kDelta) {
                        uint32_t x = acc;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
                            if (lane >= o) x += y;
                        }
                        ex = x - acc;
                        run = __shfl_sync(0xFFFFFFFFu, x, 31);
                    }
                    uint32_t* const dst = valw + Kp * lane;
#pragma unroll
                    for (int k = 0; k < 17; ++k)
                        if (k < static_cast<int>(Kp)) dst[k] = val[k] + ex;
                }
                unsigned last = 0;
                if (lane == 0) {
                    s_wcnt[i & 3][warp] = n_w;
                    s_wsum[i & 3][warp] = run;
                    __threadfence_block();
                    last = atomicAdd(&s_arr[i & 3], 1u) == kV3Workers - 1;
                }
                __syncwarp();
                nb_arrive(kBarAgg0 + (i & 1), kV3Threads);  // the lookback warp needs only the shared totals
                if (__shfl_sync(0xFFFFFFFFu, last, 0)) {
                    // last warp of the tile: publish the tile and group aggregates
                    // here, independent of how far the lookback warp has got
                    __threadfence_block();
                    const unsigned c = lane < kV3Workers ? *static_cast<volatile unsigned*>(&s_wcnt[i & 3][lane]) : 0u;
                    const uint32_t sm = lane < kV3Workers ? *static_cast<volatile uint32_t*>(&s_wsum[i & 3][lane]) : 0u;
                    const unsigned n_tile = __reduce_add_sync(0xFFFFFFFFu, c);
                    const uint32_t ts = __reduce_add_sync(0xFFFFFFFFu, sm);
                    const uint32_t t_sum = t == 0 ? static_cast<uint32_t>(prev_of(P) + ts) : ts;
                    if (lane == 0) {
                        s_arr[i & 3] = 0;
                        MVB_T3(t, 2);
                    }
                    publish_agg_pair(W, t, n_tile, t_sum, epoch, lane, kDelta ? 2 : 1);
                    if (lane == 0 && P.trace) {
                        MVB_T3(t, 3);
                        unsigned smid;
                        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                        P.trace[static_cast<unsigned long long>(t) * 8 + 7] =
                            (static_cast<unsigned long long>(smid) << 32) | blockIdx.x;
                    }
                }
            }
        }
    }

    // ---- completion; the last CTA produces the DecodeResult ----
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        s_last = atomicAdd(&P.hdr->done, 1ull) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    for (long long k = tid; k < W.n_groups; k += kV3Threads) {
        W.a1cnt[k] = 0;
        W.a1sum[k] = 0;
    }
    for (long long k = tid; k < W.n_super; k += kV3Threads) {
        W.a2cnt[k] = 0;
        W.a2sum[k] = 0;
    }
    Params Pf = P;
    Pf.n_groups = 0;  // (the two-level accumulators are not used here)
    finalize_pipelined(Pf, epoch, tid, reinterpret_cast<unsigned*>(smem + kS3V),
                       reinterpret_cast<long long*>(smem + kS3EP));
}

#undef MVB_T3

}  // namespace mvbk
