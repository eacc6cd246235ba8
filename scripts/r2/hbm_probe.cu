// HBM ceiling probe for the decode's traffic mix: read R bytes, write W bytes
// (W/R ~ 4 for c4), uint4 accesses, grid-stride.  Built by scripts/r2/hbm_probe.sh.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__global__ void expand(const uint4* __restrict__ in, uint4* __restrict__ out, size_t n_in, int ratio, int cs) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
    for (; i < n_in; i += st) {
        uint4 v = in[i];
        for (int k = 0; k < ratio; ++k) {
            uint4 o = make_uint4(v.x + k, v.y, v.z, v.w);
            uint4* p = out + (size_t)k * n_in + i;
            if (cs) __stcs(p, o); else *p = o;
        }
    }
}
__global__ void wonly(uint4* __restrict__ out, size_t n, int cs) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
    for (; i < n; i += st) { uint4 o = make_uint4(i, 0, 0, 0); if (cs) __stcs(out + i, o); else out[i] = o; }
}
int main() {
    const size_t R = 1095ull << 20, W = 4ull * R;
    uint4 *in, *out;
    cudaMalloc(&in, R); cudaMalloc(&out, W);
    cudaMemset(in, 1, R); cudaMemset(out, 0, W);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int cs = 0; cs < 2; ++cs)
    for (int bl = 2; bl <= 16; bl *= 2) {
        float best = 1e9;
        for (int r = 0; r < 6; ++r) {
            cudaEventRecord(a);
            expand<<<sms * bl, 256>>>(in, out, R / 16, 4, cs);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (r && ms < best) best = ms;
        }
        printf("expand r1:w4 cs=%d blocks/SM=%d: %.3f ms  %.0f GB/s\n", cs, bl, best, (R + W) / best / 1e6);
    }
    for (int cs = 0; cs < 2; ++cs) {
        float best = 1e9;
        for (int r = 0; r < 6; ++r) {
            cudaEventRecord(a);
            wonly<<<sms * 8, 256>>>(out, W / 16, cs);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (r && ms < best) best = ms;
        }
        printf("write-only cs=%d: %.3f ms  %.0f GB/s\n", cs, best, W / best / 1e6);
    }
    float best = 1e9;
    for (int r = 0; r < 6; ++r) {
        cudaEventRecord(a);
        cudaMemcpyAsync(out, out + W / 32, W / 2, cudaMemcpyDeviceToDevice);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (r && ms < best) best = ms;
    }
    printf("memcpy d2d %zu MB: %.3f ms  %.0f GB/s (r+w)\n", W / 2 >> 20, best, W / best / 1e6);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
