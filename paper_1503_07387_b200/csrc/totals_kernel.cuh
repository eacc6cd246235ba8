// totals_kernel.cuh -- the seam fix-up of the sharded delta decode.
//
// Each GPU needs the total of the gaps of every earlier shard before it can
// emit absolute values (the decomposition of vbyte.cpp:63-74's running
// `prev += value` into per-shard partial sums).  The totals themselves come
// from the single-read decoder's totals pass (decode_fused.cuh, mode 1);
// this kernel turns the all-gathered records into one shard's carry.
#pragma once

#include "decode_kernel.cuh"

namespace mvbk {

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
