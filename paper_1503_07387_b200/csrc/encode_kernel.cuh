// encode_kernel.cuh -- device-side VByte encoder.
//
// The write side of the same format: encode_sequence / encode_deltas
// (/root/reference/proj/core/src/vbyte.cpp:17-45, delta_encode :76-86) as
// three kernels over tiles of 4096 values:
//   1. vbyte_enc_sizes: per-tile encoded byte count (encoded_size,
//      vbyte.cpp:9-15); for deltas the gaps x[i] - x[i-1] (x[-1] = 0) and the
//      first index where the input decreases (the reference throws
//      std::invalid_argument there, vbyte.cpp:80-81);
//   2. vbyte_enc_scan: exclusive scan of the tile byte counts (one CTA) and the
//      total length;
//   3. vbyte_enc_write: per-tile block scan of the value sizes and the bytes
//      (7-bit groups LSB first, continuation bit on all but the last,
//      vbyte.cpp:17-25) written at their offsets.
#pragma once

#include <cstdint>

namespace mvbk {

constexpr int kEncThreads = 256;
constexpr int kEncPer = 16;                      // values per thread
constexpr int kEncTile = kEncThreads * kEncPer;  // 4096 values per tile

__device__ __forceinline__ uint32_t enc_size(uint32_t x) {
    return 1u + (x >= (1u << 7)) + (x >= (1u << 14)) + (x >= (1u << 21)) + (x >= (1u << 28));
}

template <bool kDelta>
__device__ __forceinline__ uint32_t enc_value(const uint32_t* v, unsigned long long i) {
    if (!kDelta) return v[i];
    return v[i] - (i ? v[i - 1] : 0u);
}

template <bool kDelta>
__global__ void __launch_bounds__(kEncThreads) vbyte_enc_sizes(const uint32_t* v, unsigned long long n,
                                                              unsigned long long* tile_bytes,
                                                              unsigned long long* bad_index) {
    __shared__ unsigned long long s_w[kEncThreads / 32];
    const unsigned long long i0 = static_cast<unsigned long long>(blockIdx.x) * kEncTile + threadIdx.x * kEncPer;
    unsigned long long bytes = 0;
#pragma unroll
    for (int k = 0; k < kEncPer; ++k) {
        const unsigned long long i = i0 + k;
        if (i < n) {
            bytes += enc_size(enc_value<kDelta>(v, i));
            if (kDelta && i && v[i] < v[i - 1]) atomicMin(bad_index, i);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xFFFFFFFFu, bytes, o);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = bytes;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int k = 0; k < kEncThreads / 32; ++k) t += s_w[k];
        tile_bytes[blockIdx.x] = t;
    }
}

// Exclusive scan of n_tiles tile byte counts in place; total -> *total.
__global__ void __launch_bounds__(1024) vbyte_enc_scan(unsigned long long* tile_bytes, unsigned long long n_tiles,
                                                       unsigned long long* total) {
    __shared__ unsigned long long s_w[32];
    __shared__ unsigned long long s_carry;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (unsigned long long b = 0; b < n_tiles; b += 1024) {
        const unsigned long long i = b + threadIdx.x;
        const unsigned long long x = i < n_tiles ? tile_bytes[i] : 0ull;
        unsigned long long incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_w[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            unsigned long long w = s_w[lane];
            unsigned long long wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, wi, o);
                if (lane >= o) wi += y;
            }
            s_w[lane] = wi - w;  // exclusive warp offsets
        }
        __syncthreads();
        const unsigned long long carry = s_carry;
        if (i < n_tiles) tile_bytes[i] = carry + s_w[wid] + incl - x;
        __syncthreads();
        if (threadIdx.x == 1023) s_carry = carry + s_w[wid] + incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = s_carry;
}

template <bool kDelta>
__global__ void __launch_bounds__(kEncThreads) vbyte_enc_write(const uint32_t* v, unsigned long long n,
                                                              const unsigned long long* tile_off, uint8_t* out) {
    // The tile's bytes are assembled in shared memory at the same offset modulo 16
    // as their place in `out`, then copied out as aligned 16-byte chunks (the
    // ragged first and last chunk byte by byte): the threads' runs of 16..80
    // bytes never go to global memory one byte at a time.
    __shared__ __align__(16) uint8_t s_out[kEncTile * 5 + 32];
    __shared__ unsigned long long s_w[kEncThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned long long i0 = static_cast<unsigned long long>(blockIdx.x) * kEncTile + threadIdx.x * kEncPer;
    uint32_t x[kEncPer];
    unsigned long long bytes = 0;
    if (i0 + kEncPer <= n && !kDelta && (reinterpret_cast<uintptr_t>(v) & 15u) == 0u) {
        // (a thread's 16 values are 64 contiguous bytes, 16-byte aligned if v is)
        const uint4* q = reinterpret_cast<const uint4*>(v + i0);
#pragma unroll
        for (int k = 0; k < kEncPer / 4; ++k) {
            const uint4 t = __ldg(q + k);
            x[4 * k] = t.x;
            x[4 * k + 1] = t.y;
            x[4 * k + 2] = t.z;
            x[4 * k + 3] = t.w;
        }
#pragma unroll
        for (int k = 0; k < kEncPer; ++k) bytes += enc_size(x[k]);
    } else {
#pragma unroll
        for (int k = 0; k < kEncPer; ++k) {
            const unsigned long long i = i0 + k;
            x[k] = i < n ? enc_value<kDelta>(v, i) : 0u;
            bytes += i < n ? enc_size(x[k]) : 0u;
        }
    }
    unsigned long long incl = bytes;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_w[wid] = incl;
    __syncthreads();
    unsigned long long wbase = 0, total = 0;
#pragma unroll
    for (int k = 0; k < kEncThreads / 32; ++k) {
        if (k < wid) wbase += s_w[k];
        total += s_w[k];
    }
    uint8_t* const dst = out + tile_off[blockIdx.x];
    const uint32_t a = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(dst) & 15u);
    uint8_t* p = s_out + a + static_cast<uint32_t>(wbase + incl - bytes);
#pragma unroll
    for (int k = 0; k < kEncPer; ++k) {
        if (i0 + k < n) {
            uint32_t y = x[k];
            while (y >= 0x80u) {
                *p++ = static_cast<uint8_t>(y | 0x80u);
                y >>= 7;
            }
            *p++ = static_cast<uint8_t>(y);
        }
    }
    __syncthreads();
    const uint32_t end = a + static_cast<uint32_t>(total);  // s_out[a, end) <-> (dst - a)[a, end)
    uint8_t* const base = dst - a;                          // 16-byte aligned
    for (uint32_t c = threadIdx.x; 16u * c < end; c += kEncThreads) {
        const uint32_t lo = 16u * c, hi = lo + 16u;
        if (lo >= a && hi <= end) {
            *reinterpret_cast<uint4*>(base + lo) = *reinterpret_cast<const uint4*>(s_out + lo);
        } else {
            for (uint32_t b = lo > a ? lo : a; b < (hi < end ? hi : end); ++b) base[b] = s_out[b];
        }
    }
}

}  // namespace mvbk
