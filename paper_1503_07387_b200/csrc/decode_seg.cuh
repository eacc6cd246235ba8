// decode_seg.cuh -- two-kernel strict-mode decoder: segment totals, then one
// warp per segment with its output index and carry known up front.
//
// The stream (in 16-byte-aligned coordinates q = p + mis) is cut into S
// equal segments of a multiple of 512 bytes, about four per resident warp.
//
//   A. vbyte_seg_totals: one warp per segment counts the integers that END
//      in it (terminator bytes) and sums their values mod 2^32 (the totals
//      pre-pass of the sharded decode, totals_kernel.cuh), and rolls both up
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

#include "decode_pipelined.cuh"
#include "totals_kernel.cuh"

namespace mvbk {

constexpr int kSegWarps = 4;  // warps per CTA
constexpr int kSegThreads = 32 * kSegWarps;
constexpr int kSegSlice = 512;
constexpr int kSegVW = 528;   // V words per warp (8 halo + 512 + pad to 64 B)
constexpr int kSegEPH = 536;  // EP halfwords per warp: [7] previous end, [8 + k] ends, 8 padding (16-B multiple)
constexpr int kSegSmem = kSegWarps * (4 * kSegVW + 2 * kSegEPH);
static_assert((4 * kSegVW) % 64 == 0 && (2 * kSegEPH) % 16 == 0, "alignment");

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
    WsHeader* hdr;
    mvb_result* res_dev;
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

// ------------------------------------------------------------------ kernel A

template <bool kDelta>
__global__ void __launch_bounds__(kSegThreads) vbyte_seg_totals(SegParams S) {
    const int lane = threadIdx.x & 31;
    const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    for (long long s = gw; s < S.n_seg; s += nw) {
        const long long qs = s * S.seg_bytes;
        const long long qe = qs + S.seg_bytes;
        // previous 8 bytes of the first slice (lane 0)
        uint32_t pw2 = 0, pw3 = 0;
        if (lane == 0) {
            if (seg_inside(S, qs - 8, 8)) {
                const uint2 v = __ldg(reinterpret_cast<const uint2*>(S.in - S.mis + qs - 8));
                pw2 = v.x;
                pw3 = v.y;
            } else {
                pw2 = seg_word(S, qs - 8);
                pw3 = seg_word(S, qs - 4);
            }
        }
        unsigned cnt = 0;
        uint32_t sum = 0;
        for (long long q = qs; q < qe; q += kSegSlice) {
            const long long q0 = q + 16 * lane;
            const uint4 x = seg_load16(S, q0);
            const uint32_t w[4] = {x.x, x.y, x.z, x.w};
            uint32_t wp2 = __shfl_up_sync(0xFFFFFFFFu, x.z, 1), wp3 = __shfl_up_sync(0xFFFFFFFFu, x.w, 1);
            uint32_t wn = __shfl_down_sync(0xFFFFFFFFu, x.x, 1);
            const uint32_t l2 = __shfl_sync(0xFFFFFFFFu, x.z, 31), l3 = __shfl_sync(0xFFFFFFFFu, x.w, 31);
            if (lane == 0) {
                wp2 = pw2;
                wp3 = pw3;
            }
            if (lane == 31) wn = seg_inside(S, q0 + 16, 4) ? __ldg(reinterpret_cast<const uint32_t*>(S.in - S.mis + q0 + 16))
                                                           : seg_word(S, q0 + 16);
            pw2 = l2;
            pw3 = l3;
            const uint32_t T16 = hibits16(~w[0], ~w[1], ~w[2], ~w[3]);
            const uint32_t Tx = (hibits4(~wp2) | (hibits4(~wp3) << 4)) | (T16 << 8) | (hibits4(~wn) << 24);
            uint32_t ends = T16 & seg_inr16(S, q0);
            cnt += __popc(ends);
            if (kDelta) {
                const uint32_t single = ends & (Tx >> 7);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t m = (single >> (4 * k)) & 0xFu;
                    sum = __dp4a(w[k] & (((m * 0x204081u) & 0x01010101u) * 0xFFu), 0x01010101u, sum);
                }
                ends &= ~single;
                if (ends) {
                    const uint32_t d[6] = {digits4(wp2), digits4(wp3), digits4(w[0]), digits4(w[1]), digits4(w[2]),
                                           digits4(w[3])};
                    while (ends) {
                        const int j = __ffs(ends) - 1;
                        ends &= ends - 1;
                        sum += value_ending_at(j, Tx, d);
                    }
                }
            }
        }
        cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
        if (kDelta) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
        }
        if (lane == 0) {
            S.scnt[s] = cnt;
            atomicAdd(S.gcnt + (s >> 5), static_cast<unsigned long long>(cnt));
            if (kDelta) {
                S.ssum[s] = sum;
                atomicAdd(S.gsum + (s >> 5), static_cast<unsigned long long>(sum));
            }
        }
    }
}

// ------------------------------------------------------------------ kernel B

template <bool kDelta>
__global__ void __launch_bounds__(kSegThreads) vbyte_seg_decode(SegParams S) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ bool s_last;
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    char* const vbase = reinterpret_cast<char*>(smem) + wid * (4 * kSegVW);
    uint16_t* const eph = reinterpret_cast<uint16_t*>(smem + kSegWarps * 4 * kSegVW) + wid * kSegEPH;
    const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    const uint32_t r0 = 8u + 16u * static_cast<uint32_t>(lane);  // V index of this lane's chunk
    const uintptr_t out_w = reinterpret_cast<uintptr_t>(S.out) >> 2;

    for (long long s = gw; s < S.n_seg; s += nw) {
        // ---- output index and carry of the segment: groups before + segments before in the group ----
        unsigned long long base = 0;
        unsigned long long csum = 0;
        const long long g = s >> 5;
        for (long long k = lane; k < g; k += 32) {
            base += S.gcnt[k];
            if (kDelta) csum += S.gsum[k];
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
        uint32_t carry = kDelta ? static_cast<uint32_t>(csum) + (S.prev_dev ? S.prev + *S.prev_dev : S.prev) : 0u;
        unsigned long long run = base;  // output index of the next integer
        if (run >= S.count) continue;   // nothing of this segment is stored (warp-uniform)

        const long long qs = s * S.seg_bytes;
        const long long qe = qs + S.seg_bytes;
        uint32_t pw2 = 0, pw3 = 0;
        if (lane == 0) {
            if (seg_inside(S, qs - 8, 8)) {
                const uint2 v = __ldg(reinterpret_cast<const uint2*>(S.in - S.mis + qs - 8));
                pw2 = v.x;
                pw3 = v.y;
            } else {
                pw2 = seg_word(S, qs - 8);
                pw3 = seg_word(S, qs - 4);
            }
        }
        uint4 nx = seg_load16(S, qs + 16 * lane);  // prefetched slice
        long long last_end = -1;                   // stream position after the segment's last integer
        for (long long q = qs; q < qe; q += kSegSlice) {
            const long long q0 = q + 16 * lane;
            const uint4 x = nx;
            if (q + kSegSlice < qe) nx = seg_load16(S, q0 + kSegSlice);
            const uint32_t w0 = x.x, w1 = x.y, w2 = x.z, w3 = x.w;
            uint32_t wp2 = __shfl_up_sync(0xFFFFFFFFu, w2, 1), wp3 = __shfl_up_sync(0xFFFFFFFFu, w3, 1);
            uint32_t wn = __shfl_down_sync(0xFFFFFFFFu, w0, 1);
            const uint32_t l2 = __shfl_sync(0xFFFFFFFFu, w2, 31), l3 = __shfl_sync(0xFFFFFFFFu, w3, 31);
            const uint32_t nf = __shfl_sync(0xFFFFFFFFu, nx.x, 0);  // first word of the next slice
            if (lane == 0) {
                wp2 = pw2;
                wp3 = pw3;
            }
            if (lane == 31)
                wn = (q + kSegSlice < qe) ? nf
                     : seg_inside(S, q0 + 16, 4) ? __ldg(reinterpret_cast<const uint32_t*>(S.in - S.mis + q0 + 16))
                                                 : seg_word(S, q0 + 16);
            pw2 = l2;
            pw3 = l3;

            // ---- phase 1: terminators, counts ----
            const uint32_t T16 = hibits16(~w0, ~w1, ~w2, ~w3);
            const uint32_t Tx = (hibits4(~wp2) | (hibits4(~wp3) << 4)) | (T16 << 8) | (hibits4(~wn) << 24);
            const uint32_t Cx = ~Tx & 0x0FFFFFFFu;
            const uint32_t inr16 = seg_inr16(S, q0);
            const uint32_t ends16 = T16 & inr16;
            const uint32_t n_own = __popc(ends16);
            uint32_t incl = n_own;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= o) incl += y;
            }
            const uint32_t n_w = __shfl_sync(0xFFFFFFFFu, incl, 31);
            const uint32_t wexcl = incl - n_own;
            // strict: a fifth byte >= 0x10 (4 continuation bytes after an integer end)
            if (Cx & (Cx >> 1) & (Cx >> 2) & (Cx >> 3)) {
                const uint32_t five = (Tx >> 3) & (Cx >> 4) & (Cx >> 5) & (Cx >> 6) & (Cx >> 7) & inr16;
                if (five) {
                    const uint32_t g0 = w0 | (w0 << 1) | (w0 << 2) | (w0 << 3);
                    const uint32_t g1 = w1 | (w1 << 1) | (w1 << 2) | (w1 << 3);
                    const uint32_t g2 = w2 | (w2 << 1) | (w2 << 2) | (w2 << 3);
                    const uint32_t g3 = w3 | (w3 << 1) | (w3 << 2) | (w3 << 3);
                    const uint32_t bad16 = five & hibits16(g0, g1, g2, g3);
                    if (bad16) {
                        const int j = __ffs(bad16) - 1;
                        const unsigned long long idx = run + wexcl + __popc(ends16 & ((1u << j) - 1u));
                        if (idx < S.count) {
                            atomicMax(&S.hdr->err_idx_inv, ~idx);
                            atomicMax(&S.hdr->err_pos_inv, ~static_cast<unsigned long long>(q0 + j - 4 - S.mis));
                        }
                    }
                }
            }
            if (n_w == 0) continue;  // warp-uniform
            // end of integer count-1, if it ends in this slice
            if (S.count - run <= n_w && S.count - 1 - run >= wexcl && S.count - 1 - run < wexcl + n_own) {
                uint32_t m = ends16;
                for (unsigned r = static_cast<unsigned>(S.count - 1 - run - wexcl); r > 0; --r) m &= m - 1;
                S.hdr->count_end = static_cast<unsigned long long>(q0 + (__ffs(m) - 1) + 1 - S.mis);
            }
            if (wexcl + n_own == n_w && n_own) last_end = q0 + (31 - __clz(ends16)) + 1 - S.mis;

            // ---- V digit windows (positions -8 .. 511 of the slice) and EP ends ----
            const uint32_t d0 = digits4(w0), d1 = digits4(w1), d2 = digits4(w2), d3 = digits4(w3), dn = digits4(wn);
            const uint32_t vo = 4u * r0;
            *reinterpret_cast<uint4*>(vbase + v_swz(vo)) = vquad(d0, d1);
            *reinterpret_cast<uint4*>(vbase + v_swz(vo + 16)) = vquad(d1, d2);
            *reinterpret_cast<uint4*>(vbase + v_swz(vo + 32)) = vquad(d2, d3);
            *reinterpret_cast<uint4*>(vbase + v_swz(vo + 48)) = vquad(d3, dn);
            if (lane == 0) {
                const uint32_t dp2 = digits4(wp2), dp3 = digits4(wp3);
                *reinterpret_cast<uint4*>(vbase + v_swz(0)) = vquad(dp2, dp3);
                *reinterpret_cast<uint4*>(vbase + v_swz(16)) = vquad(dp3, d0);
                const uint32_t tp8 = Tx & 0xFFu;  // positions -8..-1 -> V index 0..7
                // the stream start is an integer boundary: the padding before it
                // holds no integers (they are masked out of ends16)
                eph[7] = (q <= S.mis) ? static_cast<uint16_t>(7 + (S.mis - q))
                                      : static_cast<uint16_t>(tp8 ? 31 - __clz(tp8) : 0xFFFF);
            }
            uint16_t* ep = eph + 8 + wexcl;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                if ((ends16 >> j) & 1u) {
                    *ep = static_cast<uint16_t>(r0 + j);
                    ++ep;
                }
            }
            if (n_own && wexcl + n_own == n_w) {  // zero-width padding for the last octet
                const uint16_t rl = static_cast<uint16_t>(r0 + (31 - __clz(ends16)));
#pragma unroll
                for (int k = 0; k < 8; ++k) ep[k] = rl;
            }
            __syncwarp();

            // ---- phase 2 and stores: 8 integers per lane per pass ----
            for (uint32_t q2 = 0; q2 < n_w; q2 += 256) {
                const uint32_t u = q2 + 8u * lane;
                uint32_t val[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) val[k] = 0;
                if (u < n_w) {
                    const uint4 ea = *reinterpret_cast<const uint4*>(eph + 8 + u);  // 8 ends
                    const uint32_t e[9] = {eph[7 + u], ea.x & 0xFFFFu, ea.x >> 16, ea.y & 0xFFFFu, ea.y >> 16,
                                           ea.z & 0xFFFFu, ea.z >> 16, ea.w & 0xFFFFu, ea.w >> 16};
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        val[k] = *reinterpret_cast<const uint32_t*>(vbase + v_swz(4u * ((e[k] + 1u) & 0xFFFFu))) &
                                 bmsk(7u * ((e[k + 1] - e[k]) & 0xFFFFu));
                }
                uint32_t ex = 0;
                if (kDelta) {
#pragma unroll
                    for (int k = 1; k < 8; ++k) val[k] += val[k - 1];
                    uint32_t xs = val[7];
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, xs, o);
                        if (lane >= o) xs += y;
                    }
                    ex = carry + xs - val[7];
                    carry += __shfl_sync(0xFFFFFFFFu, xs, 31);
#pragma unroll
                    for (int k = 0; k < 8; ++k) val[k] += ex;
                }
                const unsigned long long gi = run + q2;  // output index of this pass's first integer
                if (gi < S.count) {
                    const unsigned long long room = S.count - gi;
                    const unsigned npass = n_w - q2 < 256u ? n_w - q2 : 256u;
                    const unsigned plim = room < npass ? static_cast<unsigned>(room) : npass;
                    uint32_t* const op = S.out + gi;
                    switch ((4u - static_cast<unsigned>((out_w + gi) & 3u)) & 3u) {
                        case 0: store_octets<0>(op, val, lane, plim); break;
                        case 1: store_octets<1>(op, val, lane, plim); break;
                        case 2: store_octets<2>(op, val, lane, plim); break;
                        default: store_octets<3>(op, val, lane, plim); break;
                    }
                }
            }
            run += n_w;
            __syncwarp();  // V / EP are rewritten by the next slice
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const long long y = __shfl_xor_sync(0xFFFFFFFFu, last_end, o);
            last_end = y > last_end ? y : last_end;
        }
        if (lane == 0 && last_end >= 0) atomicMax(&S.hdr->last_end, static_cast<unsigned long long>(last_end));
    }

    // ---- completion; the last CTA produces the DecodeResult ----
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&S.hdr->done, 1ull) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // total integer count; then zero the group accumulators for the next launch
    unsigned long long tot = 0;
    for (long long k = threadIdx.x; k < S.n_grp; k += blockDim.x) tot += S.gcnt[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xFFFFFFFFu, tot, o);
    __shared__ unsigned long long s_tot[kSegWarps];
    if (lane == 0) s_tot[wid] = tot;
    __syncthreads();
    for (long long k = threadIdx.x; k < S.n_grp; k += blockDim.x) {
        S.gcnt[k] = 0;
        S.gsum[k] = 0;
    }
    if (threadIdx.x == 0) {
        unsigned long long total = 0;
        for (int k = 0; k < kSegWarps; ++k) total += s_tot[k];
        WsHeader* h = S.hdr;
        const unsigned long long err_inv = *reinterpret_cast<volatile unsigned long long*>(&h->err_idx_inv);
        const unsigned long long errpos_inv = *reinterpret_cast<volatile unsigned long long*>(&h->err_pos_inv);
        const unsigned long long last_end = *reinterpret_cast<volatile unsigned long long*>(&h->last_end);
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
        h->err_idx_inv = 0;
        h->err_pos_inv = 0;
        h->last_end = 0;
        h->count_end = 0;
        h->epoch = h->epoch + 1;
    }
    __threadfence();
}

}  // namespace mvbk
