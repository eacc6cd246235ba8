// decode_lists.cuh -- batched delta posting lists (BASELINE config 3): one
// warp per list, long lists through the fused decoder's dp2a slices.
//
// Replaces the per-list decode_delta_stream loop of the reference's batch
// runner (tools/bench/runner.cpp:28-61): every list is decoded exactly as one
// decode_delta_scalar call would (vbyte.cpp:63-74), with its own DecodeResult.
//
// Lists are handed out by a ticket counter (in `order` if given: longest
// first).  A list's bytes [lo, hi) (stream coordinates q, L.ab 16-byte
// aligned) are cut into units of kLUnit bytes from U0 = lo & ~15:
//
//   * units of four whole 992-byte slices (the last one: the whole slices left
//     before hi) arrive in shared memory by one TMA bulk
//     copy each, the next unit's while this one is decoded, and go through
//     slice_d3_odd<kCheck> (decode_fused.cuh): odd lane strides, one dp2a per
//     byte, bulk copy-out.  A list is decoded by one warp from its first byte
//     on, so its output index and delta carry are simply carried from slice
//     to slice -- no totals pass, no prefix tree.  The <= 15 bytes before the
//     list in its first unit are zeroed in shared memory (they decode as that
//     many zeros, which the first slice's copy-out skips);
//   * a slice with a byte after three continuation bytes (an integer of 4+
//     bytes, or a malformed one) or holding integer count-1 is not decoded by
//     the dp2a path: the rest of its unit goes through the general range
//     decoder (decode_range_ll16: range masks, strict checks, the end of
//     integer count-1), which starts at any 16-byte boundary -- every d3 slice
//     starts at one;
//   * the bytes after the last whole slice (under 1 KiB per list) go through
//     the general range decoder as well.
//
// The dp2a path counts every byte before a slice in its carry, the general
// path complete integers only: the partial value of the integer straddling
// the hand-over point converts one into the other.
#pragma once

#include "decode_fused.cuh"

namespace mvbk {

// A list unit is four 992-byte slices of 31-byte lanes (one slice shape: the
// kernel's hot code stays small -- with the stream decoder's 3 x 992 + 1120
// units, warps in different slice shapes and in the general path evicted each
// other's instructions: 2.5 no-instruction stalls per issued instruction).
constexpr int kLUnit = 4 * 992;
static_assert(kLUnit % 16 == 0 && kLUnit + 32 <= kUnitBuf, "list units fit the unit buffers");

template <bool kSwz>
__device__ __noinline__ void lists_range_general(const ByteRange R, long long qs, long long qe, unsigned long long base,
                                                 uint32_t carry, unsigned long long limit, uint32_t* out,
                                                 uint32_t* stage, uint32_t ring, const RangeSink K, RangeOut* ro) {
    RangeOut r;
    decode_range_ll16<true, kSwz>(R, qs, qe, base, carry, limit, out, stage, ring, threadIdx.x & 31, K, r);
    *ro = r;
}

__global__ void __launch_bounds__(kSegThreads, kFBlocks) vbyte_lists_decode_units(ListParams L) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ bool s_last;
    __shared__ unsigned long long s_err_idx[kSegWarps];
    __shared__ long long s_err_pos[kSegWarps], s_count_end[kSegWarps];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    uint8_t* const wbuf = smem + wid * kFWarpBytes;  // two unit buffers ([0, 16) the bytes before the unit), staging
    uint32_t* const stage = reinterpret_cast<uint32_t*>(wbuf + 2 * kUnitBuf);
    unsigned long long* const bar_p = reinterpret_cast<unsigned long long*>(smem + kSegWarps * kFWarpBytes) + 2 * wid;
    const uint32_t bar0 = static_cast<uint32_t>(__cvta_generic_to_shared(bar_p));
    const uint32_t buf0 = static_cast<uint32_t>(__cvta_generic_to_shared(wbuf));
    const uint32_t st_base = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
    if (lane == 0) {
        mbar_init_warp(bar_p);
        mbar_init_warp(bar_p + 1);
    }
    __syncwarp();
    uint32_t phases = 0;  // bit b: parity of buffer b's next completion
    const unsigned long long pol = l2_evict_first();
    unsigned* const ticket = reinterpret_cast<unsigned*>(&L.hdr->ticket);
    // One list of lookahead in lane 0, spread over the current list's slices so
    // that no step waits for the one before: the next ticket (taken when this
    // list starts), its list index (order[]), that list's first byte offset,
    // and an L2 prefetch of its first unit.  (Per list, the chain ticket ->
    // order -> offsets -> first bytes is four memory latencies; a warp decodes
    // ~28 lists of config 3.)
    const unsigned n_lists32 = static_cast<unsigned>(L.n_lists);
    unsigned t_nx = 0, l_nx = 0;
    unsigned long long b0_nx = 0;
    int la = 0;  // (warp-uniform) lookahead steps done for t_nx: 0 ticket taken, 1 list index loaded, 2 offset loaded, 3 prefetched
    if (lane == 0) t_nx = atomicAdd(ticket, 1u);
    auto lookahead = [&]() {  // one more step for the next list (the loads: lane 0)
        if (la >= 3) return;
        if (lane == 0 && t_nx < n_lists32) {
            if (la == 0) l_nx = L.order ? L.order[t_nx] : t_nx;
            else if (la == 1) b0_nx = L.byte_off[l_nx];
            else {
                const long long q = (L.mis0 + static_cast<long long>(b0_nx)) & ~15ll;
                const long long left = ((L.mis0 + L.in_len) & ~15ll) - q;
                if (left >= 16)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(L.ab + q),
                                 "r"(static_cast<uint32_t>(left < kLUnit ? left : kLUnit))
                                 : "memory");
            }
        }
        ++la;
    };
    while (true) {
        while (la < 2) lookahead();  // (a short previous list: finish the chain up to the list index and offset)
        const unsigned k_list = __shfl_sync(0xFFFFFFFFu, t_nx, 0);
        if (k_list >= n_lists32) break;
        const long long l = __shfl_sync(0xFFFFFFFFu, l_nx, 0);
        if (lane == 0) t_nx = atomicAdd(ticket, 1u);
        la = 0;
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
            const RangeSink K = {nullptr, &s_err_idx[wid], &s_err_pos[wid], &s_count_end[wid]};
            const unsigned long long limit = base + cnt;
            const long long U0 = R.lo & ~15ll;
            const long long span = R.hi - U0;
            // slices (the last one may be partial); a list starting in the batch's first
            // 16-byte block takes the general path (its first unit would start before `in`)
            const int n_sl = R.hi > R.lo && U0 >= R.elo ? static_cast<int>((span + 991) / 992) : 0;
            const int n_full = (n_sl + 3) / 4;                                        // units of up to four slices
            uint32_t carry = L.prev ? L.prev[l] : 0u;  // complete integers before (the general path's convention)
            unsigned long long run = base;             // the next output index
            long long last_end = -1;                   // the end of the last integer the general path saw
            long long qs = U0;                         // everything before qs is decoded
            RangeOut ro;
            // integers ending in [from, to) through the general range decoder (bytes
            // from `to` on are outside its range: an integer straddling `to` is left
            // to whoever decodes from there)
            auto general = [&](long long from, long long to, uint32_t ring) {
#if MVB_BULK_OUT
                stage_wait_read(lane);  // (the staging buffer is rewritten with generic stores)
                __syncwarp();
#endif
                const ByteRange Rs = {R.ab, R.lo, to, R.elo, R.ehi};
                lists_range_general<true>(Rs, from, to, run, carry, limit, L.out, stage, ring, K, &ro);
                run += ro.n;
                carry = ro.carry;
                if (ro.last_end >= 0) last_end = ro.last_end;
                __syncwarp();
            };
            if (n_full > 0) {
                const uint32_t stray = static_cast<uint32_t>(R.lo - U0);
                int loaded = -1, waited = -1;  // units whose load is issued / has landed
                uint32_t tma_mask = 0;  // bit b: buffer b's unit has a bulk copy to wait for
                uint32_t rem = 0;  // lane j: byte j of the loaded unit's last, partial 16-byte block
                auto wait_load = [&](int b) {
                    if ((tma_mask >> b) & 1u) {
                        while (!mbar_test(bar0 + 8u * b, (phases >> b) & 1u)) {
                        }
                        phases ^= 1u << b;
                    }
                };
                // unit k's bytes [u_lo, u_lo + ub): whole 16-byte blocks by one TMA bulk copy
                // (with the 16 bytes before the unit, except unit 0: they are zeroed), the
                // last ub % 16 bytes one per lane (the block may end outside the buffer)
                auto unit_bytes = [&](int k) -> uint32_t {
                    const long long left = span - static_cast<long long>(k) * kLUnit;
                    return static_cast<uint32_t>(left < kLUnit ? left : kLUnit);
                };
                auto load_unit = [&](int k) {
                    const int b = k & 1;
                    const uint32_t ub = unit_bytes(k), tb = ub & ~15u;
                    const uint8_t* src = R.ab + U0 + static_cast<long long>(k) * kLUnit;
                    const bool tma = k > 0 || tb > 0;  // (warp-uniform; units after the first always load their 16 bytes before)
                    tma_mask = (tma_mask & ~(1u << b)) | (tma ? 1u << b : 0u);
                    // (everything loaded lies inside the caller's buffer and the unit buffer)
                    MVB_CHECK(src >= R.ab + R.elo && src + ub <= R.ab + R.ehi && ub <= static_cast<uint32_t>(kLUnit) &&
                              (k == 0 || src - 16 >= R.ab + R.elo));
                    if (tma && lane == 0) {
                        if (k == 0) tma_bulk_load(buf0 + 16u, src, tb, bar0);
                        else tma_bulk_load(buf0 + b * kUnitBuf, src - 16, tb + 16u, bar0 + 8u * b);
                    }
                    rem = static_cast<uint32_t>(lane) < ub - tb ? src[tb + lane] : 0u;
                    loaded = k;
                };
                load_unit(0);
                for (int k = 0; k < n_full && run < limit; ++k) {
                    const int b = k & 1;
                    const uint32_t ub = unit_bytes(k);
                    const uint32_t ubuf = buf0 + b * kUnitBuf + 16u;
                    const int sl = n_sl - 4 * k < 4 ? n_sl - 4 * k : 4;  // this unit's slices
                    wait_load(b);
                    waited = k;
                    if (ub < 992u * sl) {
                        // the last slice is partial: the bytes from the list's end on are
                        // zeroed (the slice drops the integers they decode as)
                        if (lane < 16) asm volatile("st.shared.u8 [%0], %1;" ::"r"(ubuf + (ub & ~15u) + lane), "r"(rem) : "memory");
                        for (uint32_t o = ((ub + 15u) & ~15u) + 16u * lane; o < 992u * sl + 16u; o += 512u)
                            asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(ubuf + o), "r"(0u) : "memory");
                    }
                    if (k + 1 < n_full) load_unit(k + 1);
                    if (k == 0) {
                        // the 4 bytes before the unit and the bytes before the list: zeros
                        if (static_cast<uint32_t>(lane) < 4u + stray)
                            asm volatile("st.shared.u8 [%0], %1;" ::"r"(ubuf - 4u + lane), "r"(0u) : "memory");
                    }
                    __syncwarp();
                    // the dp2a path's carry counts every byte before the slice
                    uint32_t wb = 0;
                    if (k > 0) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(wb) : "r"(ubuf - 4u) : "memory");
                    uint32_t cb = carry + tail_value(wb);
                    uint32_t* op = L.out + run - (k == 0 ? stray : 0u);
                    const uint32_t* const lim = L.out + limit;
                    const long long u_lo = U0 + static_cast<long long>(k) * kLUnit;
                    int i = 0;
#pragma unroll 1
                    for (; i < sl; ++i) {
                        lookahead();
                        uint32_t end_off = 0;
                        const uint32_t pad = 992u * (i + 1) > ub ? 992u * (i + 1) - ub : 0u;  // (the unit's last slice)
                        if (!slice_d3_odd<8, true>(ubuf, 992u * i, st_base, op, cb, lane, pol,
                                                   (k == 0 && i == 0) ? stray : 0u, lim, &end_off, pad))
                            break;
                        if (end_off) {  // integer count-1 ended the slice: the list is done
                            if (lane == 0) s_count_end[wid] = u_lo + 992 * i + end_off - R.lo;
                            ++i;
                            break;
                        }
                    }
                    MVB_CHECK(op <= lim);  // (the slices stored nothing at or past integer count)
                    const uint32_t done = 992u * i;  // unit bytes decoded by slices
                    if (done > 0) {
                        // back to the general convention at u_lo + done
                        run = static_cast<unsigned long long>(op - L.out);
                        uint32_t we;  // the 4 bytes before u_lo + done (16-byte-aligned offset: an aligned word)
                        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(we) : "r"(ubuf + done - 4u) : "memory");
                        carry = cb - tail_value(we);
                    }
                    qs = u_lo + done < R.hi ? u_lo + done : R.hi;
                    if (i < sl && run < limit) {
                        // the rest of the unit through the general path (this unit's
                        // buffer is free: it reads global memory, its ring goes here)
                        const long long u_hi = u_lo + 992 * sl < R.hi ? u_lo + 992 * sl : R.hi;
                        general(qs, u_hi, buf0 + b * kUnitBuf);
                        qs = u_hi;
                    }
                }
                // (a count limit reached with the next unit's load in flight: let it land)
                for (int k = waited + 1; k <= loaded; ++k) wait_load(k & 1);
            }
            if (run < limit && qs < R.hi) general(qs, R.hi, buf0);
            __syncwarp();
            const unsigned long long n_done = run - base;
            const unsigned long long ei = s_err_idx[wid];
            if (ei != ~0ull && ei < base + cnt) {
                r.status = MVB_MALFORMED;
                r.values_written = ei - base;
                r.bytes_consumed = static_cast<unsigned long long>(s_err_pos[wid]);
            } else if (n_done >= cnt) {
                r.status = MVB_OK;
                r.values_written = cnt;
                r.bytes_consumed = static_cast<unsigned long long>(s_count_end[wid]);
            } else {
                // truncated: the end of the list's last integer -- the general path's,
                // or (it saw none) the last terminator before qs
                if (last_end < 0 && n_done > 0) {
                    long long p = qs < R.hi ? qs : R.hi;
                    while (p > R.lo && (R.ab[p - 1] & 0x80u)) --p;
                    last_end = p - R.lo;
                }
                r.status = MVB_TRUNCATED;
                r.values_written = n_done;
                r.bytes_consumed = last_end >= 0 ? static_cast<unsigned long long>(last_end) : 0ull;
            }
        }
        if (lane == 0 && L.results) L.results[l] = r;
    }
#if MVB_BULK_OUT
    stage_wait_all(lane);
#endif
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
