// decode_pipelined.cuh -- persistent, software-pipelined strict-mode decoder.
//
// Same tile algorithm as vbyte_decode_kernel (decode_kernel.cuh), restructured
// so that no CTA waits on memory latency or on the lookback:
//
//   * persistent CTAs (grid = resident capacity), tile t_i = blockIdx + i*grid;
//   * the next tile's 4 KiB (+16-byte halos) is prefetched into shared memory
//     by a 1-D TMA bulk copy (cp.async.bulk + mbarrier) while the current
//     tile is decoded;
//   * 8 worker warps decode tile t_i (phase 1, scatter, phase 2), publish its
//     count and gap-sum aggregates, and park its values (delta: in-tile
//     prefix sums) in a double-buffered shared-memory slot;
//   * a 9th "lookback" warp resolves tile t_{i-2}'s output index and carry
//     (two-level decoupled lookback).  Two iterations after publication every
//     predecessor's aggregate is normally out, so the lookback almost never
//     waits -- with a lag of one it had to wait for the slowest CTA of the
//     previous wave, which throttled the whole grid;
//   * the workers store t_{i-2}'s values (aligned 128-bit streaming stores)
//     right after the per-iteration barrier.
//
// The DecodeResult needs three stream positions (end of integer count-1, end
// of the last integer, start of the first malformed integer).  They are not
// tracked per tile: the finalizing CTA recovers them from the published tile
// prefixes and one re-scanned tile (finalize_pipelined).
//
// Replaces the reference's stream loop (/root/reference/proj/core/src/
// stream_loop.hpp:31-129) for DecodeMode::strict; semantics as in
// decode_kernel.cuh (oracle: vbyte.cpp:47-74, internal.hpp:22-37).
#pragma once

#include "decode_kernel.cuh"

namespace mvbk {

constexpr int kPWorkers = 8;                       // worker warps (256 threads, one 4 KiB tile)
constexpr int kPWorkerThreads = 32 * kPWorkers;
constexpr int kPThreads = kPWorkerThreads + 32;    // + the lookback warp
constexpr int kPLBWarp = kPWorkers;
constexpr int kInBuf = kTile + 2 * kHalo;          // tile + 16-byte halos
constexpr int kVal = kPasses * kPWorkerThreads * 8;  // 4096 values per tile slot
constexpr int kLag = 2;                            // iterations between decode and lookback
constexpr unsigned kWorkerBar = 1;                 // named barrier id for the 256 workers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(unsigned long long* b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void workers_sync() {
    asm volatile("bar.sync %0, %1;" ::"r"(kWorkerBar), "r"(kPWorkerThreads) : "memory");
}


// Bank-conflict swizzles (scripts/smem_model.py).  V holds one word per byte
// position; worker t stores its 16 words as four 16-byte chunks at a 64-byte
// stride, which without a swizzle puts 16 lanes on the same 4 banks.  XOR-ing
// word-address bits 2-3 with bits 5-6 keeps 16-byte chunks intact and spreads
// the 8 lanes of each wavefront over all 8 chunk slots.  VAL (parked values,
// two 16-byte chunks per lane) uses the 3-bit XOR of the chunk index with its
// 128-byte row, which keeps both the park stores and the copy-out's
// consecutive-chunk loads conflict-free.
__device__ __forceinline__ uint32_t v_swz(uint32_t byte_off) { return byte_off ^ ((byte_off >> 3) & 0x30u); }
__device__ __forceinline__ uint32_t val_chunk(uint32_t c) { return c ^ ((c >> 3) & 7u); }

// Tile geometry helpers.
__device__ __forceinline__ long long tile_pos0(const Params& P, long long t) { return t * kTile - P.mis; }
// Interior tiles: the whole buffer [tpos0-16, tpos0+4096+16) lies inside the stream.
__device__ __forceinline__ bool tile_interior(const Params& P, long long t) {
    const long long p = tile_pos0(P, t);
    return p - kHalo >= 0 && p + kTile + kHalo <= P.len;
}

// Integer-end mask of one 16-byte chunk at stream position p0 (strict mode:
// terminators inside [0, len)), for the finalize re-scan.
__device__ __forceinline__ uint32_t chunk_ends(const Params& P, long long p0) {
    const uint32_t w0 = word_slow(P, p0), w1 = word_slow(P, p0 + 4), w2 = word_slow(P, p0 + 8),
                   w3 = word_slow(P, p0 + 12);
    const uint32_t m = hibits16(~w0, ~w1, ~w2, ~w3);
    const long long lo = p0 < 0 ? -p0 : 0;
    const long long hi = P.len - p0 < 16 ? P.len - p0 : 16;
    const uint32_t inr = (hi <= lo) ? 0u : ((0xFFFFu >> (16 - (hi - lo))) << lo) & 0xFFFFu;
    return m & inr;
}

// Inclusive integer count through tile t (published inclusive descriptor).
__device__ __forceinline__ unsigned long long tile_incl_count(const Params& P, long long t) {
    return t < 0 ? 0ull : desc_value<false>(ld_relaxed(P.dcnt + t));
}

// Position just after the k-th (0-based) integer end of tile t, computed by
// the whole CTA (threads >= 256 only take part in the barriers).
__device__ long long tile_end_after(const Params& P, long long t, unsigned k, int tid, unsigned* s_scan,
                                    long long* s_result) {
    const long long p0 = tile_pos0(P, t) + 16ll * (tid < 256 ? tid : 0);
    const uint32_t e = tid < 256 ? chunk_ends(P, p0) : 0u;
    if (tid < 256) s_scan[tid] = __popc(e);
    __syncthreads();
    if (tid == 0) {
        unsigned acc = 0;
        for (int j = 0; j < 256; ++j) {
            const unsigned c = s_scan[j];
            s_scan[j] = acc;
            acc += c;
        }
    }
    __syncthreads();
    if (tid < 256) {
        const unsigned before = s_scan[tid];
        if (k >= before && k < before + __popc(e)) {
            uint32_t m = e;
            for (unsigned r = k - before; r > 0; --r) m &= m - 1;
            *s_result = p0 + (__ffs(m) - 1) + 1;
        }
    }
    __syncthreads();
    return *s_result;
}

// Finalize for the pipelined kernel: run by the whole last CTA once every
// tile has published its inclusive prefixes.
__device__ void finalize_pipelined(const Params& P, unsigned long long epoch, int tid, unsigned* s_scan,
                                   long long* s_result) {
    __threadfence();
    for (unsigned i = tid; i < P.n_groups; i += blockDim.x) {
        P.gacc_cnt[i] = 0;
        P.gacc_sum[i] = 0;
    }
    const long long nt = P.n_tiles;
    const unsigned long long total = tile_incl_count(P, nt - 1);
    WsHeader* h = P.hdr;
    const unsigned long long epos_inv = *reinterpret_cast<volatile unsigned long long*>(&h->err_pos_inv);
    mvb_result r;
    r.reserved = 0;
    bool done = false;
    if (epos_inv != 0ull) {
        // first malformed integer start s: its index = integer ends before s
        const long long s = static_cast<long long>(~epos_inv);
        const long long ts = (s + P.mis) / kTile;
        const unsigned long long before_tile = tile_incl_count(P, ts - 1);
        if (tid == 0) *s_result = 0;
        __syncthreads();
        if (tid < 256) {
            const long long p0 = tile_pos0(P, ts) + 16ll * tid;
            uint32_t e = chunk_ends(P, p0);
            if (p0 >= s) e = 0;
            else if (p0 + 16 > s) e &= (1u << (s - p0)) - 1u;
            if (e) atomicAdd(reinterpret_cast<unsigned long long*>(s_result), static_cast<unsigned long long>(__popc(e)));
        }
        __syncthreads();
        const unsigned long long idx = before_tile + static_cast<unsigned long long>(*s_result);
        if (idx < P.count) {
            r.status = MVB_MALFORMED;
            r.values_written = idx;
            r.bytes_consumed = static_cast<unsigned long long>(s);
            done = true;
        }
        __syncthreads();
    }
    if (!done && total >= P.count) {
        // tile holding integer count-1: first tile whose inclusive count >= count
        long long lo = 0, hi = nt - 1;
        while (lo < hi) {
            const long long mid = (lo + hi) / 2;
            if (tile_incl_count(P, mid) >= P.count) hi = mid; else lo = mid + 1;
        }
        const unsigned k = static_cast<unsigned>(P.count - 1 - tile_incl_count(P, lo - 1));
        const long long end = tile_end_after(P, lo, k, tid, s_scan, s_result);
        r.status = MVB_OK;
        r.values_written = P.count;
        r.bytes_consumed = static_cast<unsigned long long>(end);
    } else if (!done) {
        // truncated: end of the last integer, if any
        long long tl = nt - 1;
        while (tl >= 0 && tile_incl_count(P, tl) == tile_incl_count(P, tl - 1)) --tl;
        long long end = 0;
        if (tl >= 0) {
            const unsigned k = static_cast<unsigned>(tile_incl_count(P, tl) - tile_incl_count(P, tl - 1) - 1);
            end = tile_end_after(P, tl, k, tid, s_scan, s_result);
        }
        r.status = MVB_TRUNCATED;
        r.values_written = total;
        r.bytes_consumed = static_cast<unsigned long long>(end);
    }
    if (tid == 0) {
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

// Dynamic shared memory layout of the pipelined kernel (bytes).
constexpr int kSmemIn = 0;                                   // 2 x kInBuf input buffers
constexpr int kSmemV = kSmemIn + 2 * kInBuf;                 // V[kV]
constexpr int kSmemEP = kSmemV + 4 * kV;                     // EPw[kEPw]
constexpr int kSmemVal = (kSmemEP + 4 * kEPw + 15) / 16 * 16;  // VAL[2][kVal]
constexpr int kSmemBytes = kSmemVal + 2 * 4 * kVal;
static_assert(kSmemIn % 16 == 0 && kSmemV % 16 == 0 && kSmemEP % 16 == 0, "16-byte aligned regions");

template <bool kDelta, bool kTrace>
__global__ void __launch_bounds__(kPThreads, 3) vbyte_decode_pipelined(Params P) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t (*IN)[kInBuf] = reinterpret_cast<uint8_t (*)[kInBuf]>(smem + kSmemIn);
    uint32_t* const V = reinterpret_cast<uint32_t*>(smem + kSmemV);
    uint32_t* const EPw = reinterpret_cast<uint32_t*>(smem + kSmemEP);
    uint32_t (*VAL)[kVal] = reinterpret_cast<uint32_t (*)[kVal]>(smem + kSmemVal);
    __shared__ __align__(8) unsigned long long bar[2];
    __shared__ unsigned s_warp_cnt[kPWorkers];
    __shared__ uint32_t s_pass_sum[kPasses * kPWorkers];
    __shared__ unsigned long long s_cnt_pre[4];  // indexed by the tile's iteration & 3
    __shared__ uint32_t s_sum_pre[4];
    __shared__ unsigned s_ntile[4];
    __shared__ uint32_t s_tsum[4];
    __shared__ bool s_last;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const long long G = gridDim.x;
    const long long b0 = blockIdx.x;
    const int my_tiles = static_cast<int>((static_cast<long long>(P.n_tiles) - b0 + G - 1) / G);
    const unsigned long long epoch = P.hdr->epoch + 1;  // constant during a launch
    constexpr uint32_t kStep = (4u << 16) | 7u;         // packed EPw increment per byte position
    const int lp0 = kHalo + tid * kChunk;                // local coordinate of this worker's chunk
    const uint32_t x0 = static_cast<uint32_t>(lp0 + 1) * kStep;

    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kPLBWarp && lane == 0 && my_tiles > 0 && tile_interior(P, b0)) {
        mbar_expect_tx(&bar[0], kInBuf);
        tma_load_1d(IN[0], P.in + tile_pos0(P, b0) - kHalo, kInBuf, &bar[0]);
    }

    // TMA completions consumed so far per input buffer (mbarrier phase parity);
    // tile_interior() is a pure function of t, so every thread tracks it alike.
    unsigned uses0 = 0, uses1 = 0;
    unsigned ntile_lag0 = 0, ntile_lag1 = 0;  // workers: tile counts of t_{i-1}, t_{i-2}

    for (int i = 0; i < my_tiles + kLag; ++i) {
        const bool have_cur = i < my_tiles;
        const long long t = b0 + i * G;  // current tile (valid if have_cur)
        const int cb = i & 1;            // input / VAL buffer parity

        if (warp == kPLBWarp) {
            // ---- prefetch t_{i+1}; resolve t_{i-2} ----
            if (lane == 0 && i + 1 < my_tiles && tile_interior(P, t + G)) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&bar[cb ^ 1], kInBuf);
                tma_load_1d(IN[cb ^ 1], P.in + tile_pos0(P, t + G) - kHalo, kInBuf, &bar[cb ^ 1]);
            }
            // t_{i-2} was finished by the workers before barrier #1 of iteration
            // i-1, which this warp has passed: its slots and aggregates are out.
            if (i >= kLag) {
                const long long tp = t - kLag * G;
                const int ps = (i - kLag) & 3;
                const unsigned nt = s_ntile[ps];
                unsigned long long c = 0;
                uint32_t cs = prev_of(P);
                if (tp > 0) {
                    if (kDelta) {
                        lookback2_cnt_sum(P, tp, epoch, lane, &c, &cs);
                        if (lane == 0)
                            publish_inclusive<true>(P.dsum, P.gsum, tp, P.n_tiles,
                                                    static_cast<uint32_t>(cs + s_tsum[ps]), epoch);
                    } else {
                        c = lookback2<OP_SUM40>(P.dcnt, P.gcnt, tp, epoch, lane);
                    }
                    if (lane == 0) publish_inclusive<false>(P.dcnt, P.gcnt, tp, P.n_tiles, c + nt, epoch);
                }
                if (lane == 0) {
                    s_cnt_pre[ps] = c;
                    s_sum_pre[ps] = cs;
                    if (kTrace) P.trace[static_cast<unsigned long long>(tp) * 8 + 5] = gtimer();
                }
            }
        }

        // ---- workers: phase 1 of t_i ----
        uint32_t ends16 = 0, n_own = 0, incl = 0, Tx = 0;
        uint32_t w0 = 0, w1 = 0, w2 = 0, w3 = 0, wp2 = 0, wp3 = 0, wn = 0;
        if (warp < kPWorkers && have_cur) {
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
                for (int k = tid; k < kInBuf; k += kPWorkerThreads) wbuf[k] = static_cast<uint8_t>(byte_at(P, base + k));
                workers_sync();
            }
            if (kTrace && tid == 0) P.trace[static_cast<unsigned long long>(t) * 8 + 0] = gtimer();
            const uint4 q = *reinterpret_cast<const uint4*>(buf + lp0);
            w0 = q.x; w1 = q.y; w2 = q.z; w3 = q.w;
            // halo words from the neighbouring lanes (strided loads would hit 2 banks)
            wp2 = __shfl_up_sync(0xFFFFFFFFu, w2, 1);
            wp3 = __shfl_up_sync(0xFFFFFFFFu, w3, 1);
            wn = __shfl_down_sync(0xFFFFFFFFu, w0, 1);
            if (lane == 0) {
                const uint2 pv = *reinterpret_cast<const uint2*>(buf + lp0 - 8);
                wp2 = pv.x; wp3 = pv.y;
            }
            if (lane == 31) wn = *reinterpret_cast<const uint32_t*>(buf + lp0 + kChunk);

            const uint32_t T16 = hibits16(~w0, ~w1, ~w2, ~w3);
            Tx = (hibits4(~wp2) | (hibits4(~wp3) << 4)) | (T16 << 8) | (hibits4(~wn) << 24);
            const uint32_t Cx = ~Tx & 0x0FFFFFFFu;
            uint32_t inr16 = 0xFFFFu;
            if (!interior) {
                const long long p0 = tile_pos0(P, t) + static_cast<long long>(tid) * kChunk;
                const long long lo = p0 < 0 ? -p0 : 0;
                const long long hi = P.len - p0 < 16 ? P.len - p0 : 16;
                inr16 = (hi <= lo) ? 0u : ((0xFFFFu >> (16 - (hi - lo))) << lo) & 0xFFFFu;
            }
            ends16 = T16 & inr16;
            const uint32_t five = (Tx >> 3) & (Cx >> 4) & (Cx >> 5) & (Cx >> 6) & (Cx >> 7) & inr16;
            if (five) {
                const uint32_t g0 = w0 | (w0 << 1) | (w0 << 2) | (w0 << 3);
                const uint32_t g1 = w1 | (w1 << 1) | (w1 << 2) | (w1 << 3);
                const uint32_t g2 = w2 | (w2 << 1) | (w2 << 2) | (w2 << 3);
                const uint32_t g3 = w3 | (w3 << 1) | (w3 << 2) | (w3 << 3);
                const uint32_t bad16 = five & hibits16(g0, g1, g2, g3);
                if (bad16) {  // start of a malformed integer: s = p - 4 (index recovered at finalize)
                    const long long s = tile_pos0(P, t) + static_cast<long long>(tid) * kChunk + (__ffs(bad16) - 1) - 4;
                    atomicMax(&P.hdr->err_pos_inv, ~static_cast<unsigned long long>(s));
                }
            }
            n_own = __popc(ends16);
            incl = n_own;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) s_warp_cnt[warp] = incl;
        }
        __syncthreads();  // bar #1: t_i counts; t_{i-2} resolved by the lookback warp
        if (warp == kPLBWarp) continue;

        // ---- workers: store t_{i-2}: one thread per 16-byte-aligned output quad ----
        if (i >= kLag) {
            const int ps = (i - kLag) & 3;
            const unsigned long long cnt_prefix = s_cnt_pre[ps];
            const uint32_t carry = kDelta ? s_sum_pre[ps] : 0u;
            const unsigned long long room = P.count > cnt_prefix ? P.count - cnt_prefix : 0ull;
            const unsigned lim = room < ntile_lag1 ? static_cast<unsigned>(room) : ntile_lag1;
            // head: h ints up to the first 16-byte-aligned output address,
            // body: aligned quads, tail: the rest (h, tail stored singly)
            const unsigned a = static_cast<unsigned>(((reinterpret_cast<uintptr_t>(P.out) >> 2) + cnt_prefix) & 3u);
            const unsigned h = (4u - a) & 3u;
            const uint4* vq = reinterpret_cast<const uint4*>(VAL[cb]);  // (i - 2) & 1 == i & 1
            const uint32_t* vs = VAL[cb];
            uint32_t* const o = P.out + cnt_prefix;
            const unsigned hh = h < lim ? h : lim;
            const unsigned nbody = (lim - hh) >> 2;
            const unsigned tail0 = hh + 4 * nbody;
            if (tid < hh) {
                const unsigned i0 = tid;
                stg_stream4(o + i0, vs[4 * val_chunk(i0 >> 2) + (i0 & 3)] + carry);
            } else if (tid >= 4 && tid - 4 < lim - tail0) {
                const unsigned i0 = tail0 + tid - 4;
                stg_stream4(o + i0, vs[4 * val_chunk(i0 >> 2) + (i0 & 3)] + carry);
            }
            // body quad m covers tile ints h + 4m .. h + 4m + 3: chunks m, m+1 when h > 0
#define MVB_BODY(H)                                                                                   \
    for (unsigned m = tid; m < nbody; m += kPWorkerThreads) {                                         \
        uint4 x = vq[val_chunk(m)];                                                                   \
        uint32_t r0, r1, r2, r3;                                                                      \
        if (H == 0) {                                                                                 \
            r0 = x.x; r1 = x.y; r2 = x.z; r3 = x.w;                                                   \
        } else {                                                                                      \
            const uint4 y = vq[val_chunk(m + 1)];                                                     \
            if (H == 1) { r0 = x.y; r1 = x.z; r2 = x.w; r3 = y.x; }                                   \
            else if (H == 2) { r0 = x.z; r1 = x.w; r2 = y.x; r3 = y.y; }                              \
            else { r0 = x.w; r1 = y.x; r2 = y.y; r3 = y.z; }                                          \
        }                                                                                             \
        stg_stream16(o + hh + 4 * m, r0 + carry, r1 + carry, r2 + carry, r3 + carry);                 \
    }
            // h < lim implies hh == h; otherwise nbody == 0 and the body is empty
            switch (h) {
                case 0: MVB_BODY(0) break;
                case 1: MVB_BODY(1) break;
                case 2: MVB_BODY(2) break;
                default: MVB_BODY(3) break;
            }
#undef MVB_BODY
            if (kTrace && tid == 0) P.trace[static_cast<unsigned long long>(t - kLag * G) * 8 + 6] = gtimer();
        }
        ntile_lag1 = ntile_lag0;
        if (!have_cur) continue;

        // ---- workers: count aggregate, V, scatter of t_i ----
        unsigned wbase = 0, n_tile = 0;
#pragma unroll
        for (int k = 0; k < kPWorkers; ++k) {
            const unsigned c = s_warp_cnt[k];
            wbase += (k < warp) ? c : 0u;
            n_tile += c;
        }
        ntile_lag0 = n_tile;
        const unsigned tbase = wbase + incl - n_own;
        if (tid == 0) {
            if (kTrace) P.trace[static_cast<unsigned long long>(t) * 8 + 1] = gtimer();
            publish_aggregate<false>(P.dcnt, P.gcnt, P.gacc_cnt, t, P.n_tiles, n_tile, epoch);
            s_ntile[i & 3] = n_tile;
        }
        {
            const uint32_t d0 = digits4(w0), d1 = digits4(w1), d2 = digits4(w2), d3 = digits4(w3),
                           dn = digits4(wn);
            char* const vb = reinterpret_cast<char*>(V);
            const uint32_t vo = 4u * static_cast<uint32_t>(lp0);
            *reinterpret_cast<uint4*>(vb + v_swz(vo)) = vquad(d0, d1);
            *reinterpret_cast<uint4*>(vb + v_swz(vo + 16)) = vquad(d1, d2);
            *reinterpret_cast<uint4*>(vb + v_swz(vo + 32)) = vquad(d2, d3);
            *reinterpret_cast<uint4*>(vb + v_swz(vo + 48)) = vquad(d3, dn);
            if (tid == 0) {  // halo positions -8..-1 (local 8..15)
                const uint32_t dp2 = digits4(wp2), dp3 = digits4(wp3);
                *reinterpret_cast<uint4*>(vb + v_swz(32)) = vquad(dp2, dp3);
                *reinterpret_cast<uint4*>(vb + v_swz(48)) = vquad(dp3, d0);
            }
        }
        {
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
            if (tid == 0) {
                const uint32_t tp8 = Tx & 0xFFu;  // positions -8..-1
                const unsigned prev_lp = (t == 0) ? static_cast<unsigned>(kHalo - 1 + P.mis)
                                         : tp8    ? static_cast<unsigned>(8 + 31 - __clz(tp8))
                                                  : 7u;
                EPw[3] = (prev_lp + 1) * kStep;
            }
        }
        workers_sync();  // bar #2

        // ---- workers: phase 2 of t_i ----
        uint32_t val[kPasses][8];
        uint32_t lane_excl[kPasses];
#pragma unroll
        for (int p = 0; p < kPasses; ++p) {
            const unsigned u = tid + kPWorkerThreads * p;
            lane_excl[p] = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) val[p][k] = 0;
            if (8u * (kPWorkerThreads * p + 32 * warp) >= n_tile) continue;  // warp-uniform: no ints here
            if (8 * u < n_tile) {
                const uint4 qa = *reinterpret_cast<const uint4*>(EPw + 4 + 8 * u);
                const uint4 qb = *reinterpret_cast<const uint4*>(EPw + 8 + 8 * u);
                const uint32_t xs[9] = {EPw[3 + 8 * u], qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    val[p][k] = lds_at(V, v_swz(xs[k] >> 16)) & bmsk((xs[k + 1] - xs[k]) & 0xFFFFu);
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
                if (lane == 31) s_pass_sum[p * kPWorkers + warp] = x;
            }
        }
        if (kTrace && tid == 0) P.trace[static_cast<unsigned long long>(t) * 8 + 3] = gtimer();
        if (kDelta) {
            workers_sync();  // bar #3: pass sums
            const uint32_t x =
                (lane < kPasses * kPWorkers && 8u * (kPWorkerThreads * (lane / kPWorkers) + 32 * (lane % kPWorkers)) < n_tile)
                    ? s_pass_sum[lane] : 0u;
            uint32_t sc = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, sc, o);
                if (lane >= o) sc += y;
            }
            const uint32_t tile_sum = __shfl_sync(0xFFFFFFFFu, sc, 31);
#pragma unroll
            for (int p = 0; p < kPasses; ++p) lane_excl[p] += __shfl_sync(0xFFFFFFFFu, sc - x, p * kPWorkers + warp);
            if (tid == 0) {
                if (kTrace) P.trace[static_cast<unsigned long long>(t) * 8 + 4] = gtimer();
                publish_aggregate<true>(P.dsum, P.gsum, P.gacc_sum, t, P.n_tiles,
                                        t == 0 ? static_cast<uint32_t>(prev_of(P) + tile_sum) : tile_sum, epoch);
                s_tsum[i & 3] = tile_sum;
            }
        }
        // park the values (delta: in-tile inclusive prefix) until the lookback resolves t_i
        uint4* vals = reinterpret_cast<uint4*>(VAL[cb]);
#pragma unroll
        for (int p = 0; p < kPasses; ++p) {
            if (8u * (kPWorkerThreads * p + 32 * warp) >= n_tile) continue;
            const unsigned u = tid + kPWorkerThreads * p;
            const uint32_t e = lane_excl[p];
            vals[val_chunk(2 * u)] = make_uint4(val[p][0] + e, val[p][1] + e, val[p][2] + e, val[p][3] + e);
            vals[val_chunk(2 * u + 1)] = make_uint4(val[p][4] + e, val[p][5] + e, val[p][6] + e, val[p][7] + e);
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
    finalize_pipelined(P, epoch, tid, reinterpret_cast<unsigned*>(V), reinterpret_cast<long long*>(EPw));
}

}  // namespace mvbk
