// totals_kernel.cuh -- integer count and wrapping gap sum of a byte range.
//
// The pre-pass of the sharded delta decode: each GPU needs
// the total of the gaps of every earlier shard before it can emit absolute
// values, so it first reduces its own shard to (integer count, sum of values
// mod 2^32) -- the decomposition of vbyte.cpp:63-74's running `prev += value`
// into per-shard partial sums.  No output is written.  Integers are counted
// at their terminator byte, exactly like the decode kernels; the shard is
// assumed to start at an integer boundary (the decode of the same shard
// reports any malformed or truncated data with full oracle semantics).
#pragma once

#include "decode_kernel.cuh"

namespace mvbk {

// Value of the integer ending at byte j (0..15) of the 16-byte chunk w0..w3,
// given the two preceding words and the extended terminator mask Tx
// (bit x <-> chunk position x - 8).  L = distance to the previous terminator.
__device__ __forceinline__ uint32_t value_ending_at(int j, uint32_t Tx, const uint32_t (&d)[6]) {
    const uint32_t below = Tx & ((1u << (j + 8)) - 1u);
    const int L = below ? (j + 8) - (31 - __clz(below)) : 6;
    const int k = (j >> 2) + 2;                // d[] index of the word holding byte j (d[0] = word -2)
    const unsigned long long x =               // 7-bit digits of the 8 bytes of words k-1, k
        static_cast<unsigned long long>(d[k - 1]) | (static_cast<unsigned long long>(d[k]) << 28);
    const int start = 4 + (j & 3) - L + 1;     // byte offset of the integer start within those 8 bytes
    return static_cast<uint32_t>(x >> (7 * (start < 0 ? 0 : start))) & bmsk(7u * static_cast<uint32_t>(L));
}

__global__ void __launch_bounds__(kThreads) vbyte_totals_kernel(const uint8_t* in, long long mis, long long len,
                                                                unsigned n_tiles, unsigned long long* count_out,
                                                                uint32_t* sum_out) {
    __shared__ unsigned long long s_cnt[kWarps];
    __shared__ uint32_t s_sum[kWarps];
    Params P;
    P.in = in;
    P.len = len;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned long long cnt = 0;
    uint32_t sum = 0;
    for (long long t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const long long p0 = t * kTile - mis + static_cast<long long>(tid) * kChunk;
        uint32_t w[4], wp2, wp3, wn;
        const bool inside = p0 - 8 >= 0 && p0 + kChunk + 4 <= len;
        if (inside) {
            const uint4 q = ldg_stream16(in + p0);
            w[0] = q.x; w[1] = q.y; w[2] = q.z; w[3] = q.w;
            const uint2 pv = __ldg(reinterpret_cast<const uint2*>(in + p0 - 8));
            wp2 = pv.x; wp3 = pv.y;
            wn = __ldg(reinterpret_cast<const uint32_t*>(in + p0 + kChunk));
        } else {
            for (int k = 0; k < 4; ++k) w[k] = word_slow(P, p0 + 4 * k);
            wp2 = word_slow(P, p0 - 8);
            wp3 = word_slow(P, p0 - 4);
            wn = word_slow(P, p0 + 16);
        }
        const uint32_t T16 = hibits16(~w[0], ~w[1], ~w[2], ~w[3]);
        const uint32_t Tx = (hibits4(~wp2) | (hibits4(~wp3) << 4)) | (T16 << 8) | (hibits4(~wn) << 24);
        uint32_t inr16 = 0xFFFFu;
        if (!inside) {
            const long long lo = p0 < 0 ? -p0 : 0;
            const long long hi = len - p0 < 16 ? len - p0 : 16;
            inr16 = (hi <= lo) ? 0u : ((0xFFFFu >> (16 - (hi - lo))) << lo) & 0xFFFFu;
        }
        uint32_t ends = T16 & inr16;
        cnt += __popc(ends);
        // single-byte integers (terminator preceded by a terminator; bytes
        // before the range read as 0x00, a terminator): the byte is the value
        const uint32_t single = ends & (Tx >> 7);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t m = (single >> (4 * k)) & 0xFu;
            sum = __dp4a(w[k] & (((m * 0x204081u) & 0x01010101u) * 0xFFu), 0x01010101u, sum);
        }
        ends &= ~single;
        const uint32_t d[6] = {digits4(wp2), digits4(wp3), digits4(w[0]), digits4(w[1]), digits4(w[2]), digits4(w[3])};
        while (ends) {
            const int j = __ffs(ends) - 1;
            ends &= ends - 1;
            sum += value_ending_at(j, Tx, d);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
        sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
    }
    if (lane == 0) {
        s_cnt[warp] = cnt;
        s_sum[warp] = sum;
    }
    __syncthreads();
    if (tid == 0) {
        unsigned long long c = 0;
        uint32_t s = 0;
        for (int k = 0; k < kWarps; ++k) {
            c += s_cnt[k];
            s += s_sum[k];
        }
        atomicAdd(count_out, c);
        atomicAdd(sum_out, s);
    }
}

// Carry-in and output offset of shard `rank` from the all-gathered per-shard
// records (word 0 = integer count, low half of word 1 = gap sum mod 2^32):
// the exclusive scans that stitch the shards' decodes together.
__global__ void shard_carry_kernel(const unsigned long long* rec, int rank, int words, uint32_t prev,
                                   uint32_t* carry, unsigned long long* offset) {
    unsigned long long c = 0;
    uint32_t s = 0;
    for (int h = threadIdx.x; h < rank; h += 32) {
        c += rec[static_cast<long long>(h) * words];
        s += static_cast<uint32_t>(rec[static_cast<long long>(h) * words + 1]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
        s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
    }
    if (threadIdx.x == 0) {
        if (carry) *carry = prev + s;
        if (offset) *offset = c;
    }
}

}  // namespace mvbk
