// mvb_cuda.cu -- C ABI (include/mvb_cuda.h) over the sm_100a VByte kernels.
//
// Host side of the drop-in boundary.  Mirrors the reference's public decode
// entry points (/root/reference/proj/core/include/mvb/decode.hpp:42-54 and
// vbyte.hpp:51-63) and its encoder (vbyte.cpp:9-45).  There is one decode
// implementation -- the CUDA kernel -- and no CPU fallback: a missing device
// or a failed launch is reported as MVB_ERR_CUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>
#include <deque>

#include "../../include/mvb_cuda.h"
#include "decode_kernel.cuh"
#include "decode_seg.cuh"
#include <nvtx3/nvToolsExt.h>

#include "decode_fused.cuh"
#include "decode_lists.cuh"
#include "totals_kernel.cuh"
#include "encode_kernel.cuh"

#ifndef MVB_A_ITS
#define MVB_A_ITS 6  // kernel A: at least this many 1 KiB iterations per warp (c2: one wave of 6 CTAs per SM)
#endif

namespace {
// NVTX range for timeline tools; balanced on every return path.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};


using mvbk::Params;
using mvbk::WsHeader;

constexpr size_t kHeaderBytes = sizeof(WsHeader);

size_t tiles_for(size_t mis, size_t scan_len) {
    return (mis + scan_len + mvbk::kTile - 1) / mvbk::kTile;
}

size_t groups_for(size_t tiles) { return (tiles + mvbk::kGroup - 1) / mvbk::kGroup; }

// Workspace bytes for a launch of `tiles` tiles (layout in decode_kernel.cuh).
size_t ws_need(size_t tiles) {
    return kHeaderBytes + (tiles * mvbk::kDescArrays + groups_for(tiles) * mvbk::kGroupArrays) * 8;
}

// Bytes the decode of `count` integers can touch: every integer (strict or
// permissive) spans at most 5 bytes, so nothing past 5*count matters.
// Workspace layout tracking.  Every kernel family keeps its group
// accumulators zero between launches (its finalizing CTA re-zeroes them), but
// the accumulators' offset depends on the family and the launch size, so a
// launch with a different layout than the previous one on the same workspace
// could find stale descriptor words where it expects zeros.  The host
// remembers each workspace's last layout and re-zeroes the used region when
// it changes (steady-state repeated launches never pay for it).
std::mutex g_ws_mu;
std::unordered_map<const void*, unsigned long long> g_ws_layout;

cudaError_t prepare_workspace(void* ws, size_t used_bytes, unsigned long long layout, cudaStream_t s) {
    {
        std::lock_guard<std::mutex> lk(g_ws_mu);
        auto it = g_ws_layout.find(ws);
        if (it != g_ws_layout.end() && it->second == layout) return cudaSuccess;
        g_ws_layout[ws] = layout;
    }
    return cudaMemsetAsync(static_cast<char*>(ws) + kHeaderBytes, 0, used_bytes - kHeaderBytes, s);
}

size_t scan_length(size_t in_len, size_t count) {
    if (count > in_len / 5 + 1) return in_len;
    return std::min(in_len, count * 5);
}

// Strict-mode kernel: 0 the single-read fused decoder (default,
// decode_fused.cuh); 1 the per-tile kernel (decode_kernel.cuh, which serves
// permissive mode); 6 the two-kernel segmented decoder (decode_seg.cuh; the
// pipelined host drop-in's chunks use its launch pair).  Internal switch for
// tests and comparisons (mvbx_set_kernel), not part of the C ABI.
int g_kernel_choice = 0;

// Occupancy of a kernel on the current device (cached per kernel and device).
int occupancy(const void* fn, int threads, size_t smem, int* sms_out) {
    static std::mutex mu;
    static std::unordered_map<unsigned long long, int> cache;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    *sms_out = sms;
    const unsigned long long key = (reinterpret_cast<uintptr_t>(fn) << 8) ^ static_cast<unsigned long long>(dev);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
        return -1;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem) != cudaSuccess) return -1;
    if (n < 1) n = 1;
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = n;
    return n;
}

template <bool Delta, int Mode>
cudaError_t launch(const Params& p, cudaStream_t s) {
    mvbk::vbyte_decode_kernel<Delta, Mode><<<p.n_tiles, mvbk::kThreads, 0, s>>>(p);
    return cudaGetLastError();
}

// Two-kernel segmented strict decode (decode_seg.cuh): group accumulators
// zeroed, segment totals, then one warp per segment.
//
// seg_setup fills the launch parameters (segment size: about per_warp segments
// per kernel-B warp over `plan_len` bytes -- the stream, or one chunk of a
// pipelined host decode -- in whole kernel-A iterations); seg_launch_pair
// launches kernel A and kernel B (a programmatic dependent of A) over the
// segments [s_lo, s_hi).
struct SegLaunch {
    mvbk::SegParams S;
    unsigned grid_a_cap, grid_b_cap, grid_a_launch;
};


template <bool Delta>
int seg_setup(const Params& p, void* ws, size_t ws_bytes, long long plan_len, cudaStream_t s, SegLaunch& sl) {
    int sms = 0;
    const int per_sm = occupancy(reinterpret_cast<const void*>(mvbk::vbyte_seg_decode<Delta>), mvbk::kSegThreads,
                                 mvbk::kLaneSmem, &sms);
    const int per_sm_a = occupancy(reinterpret_cast<const void*>(mvbk::vbyte_seg_totals<Delta>), mvbk::kSegThreads,
                                   mvbk::kASmem, &sms);
    if (per_sm < 0 || per_sm_a < 0) return MVB_ERR_CUDA;
    const long long ctas = static_cast<long long>(per_sm) * sms;
    const long long warps = ctas * (mvbk::kSegThreads / 32);
    const long long qlen = p.mis + p.len;
    // segments per kernel-B warp: LL decodes a balanced contiguous run of them per
    // warp (finer is better balanced), V/EP hands them out round-robin
    // segments per kernel-B warp: LL decodes a static run and then pool segments
    // (about 32 segments per warp: 1 KiB on c2), V/EP hands them out round-robin
    long long seg;
    {
        const long long per_warp = 1;  // one segment (a balanced byte range) per warp
        seg = (plan_len + per_warp * warps - 1) / (per_warp * warps);
        seg = (seg + mvbk::kSegASlice - 1) / mvbk::kSegASlice * mvbk::kSegASlice;  // kernel A: whole iterations
        if (seg < mvbk::kSegASlice) seg = mvbk::kSegASlice;
    }
    const long long n_seg = (qlen + seg - 1) / seg;
    const long long n_grp = (n_seg + 31) / 32;
    const long long n_sup = (n_grp + 31) / 32;
    const size_t need = kHeaderBytes + 8 * static_cast<size_t>(n_seg) + 16 * static_cast<size_t>(n_grp) +
                        16 * static_cast<size_t>(n_sup);
    if (ws_bytes < need) return MVB_ERR_WORKSPACE;
    mvbk::SegParams& S = sl.S;
    S.in = p.in;
    S.mis = p.mis;
    S.len = p.len;
    S.count = p.count;
    S.out = p.out;
    S.prev = p.prev;
    S.prev_dev = p.prev_dev;
    S.seg_bytes = seg;
    S.n_seg = n_seg;
    S.n_grp = n_grp;
    char* b = static_cast<char*>(ws) + kHeaderBytes;
    S.gcnt = reinterpret_cast<unsigned long long*>(b);
    S.gsum = S.gcnt + n_grp;
    S.ucnt = S.gsum + n_grp;
    S.usum = S.ucnt + n_sup;
    S.n_sup = n_sup;
    S.scnt = reinterpret_cast<unsigned*>(S.usum + n_sup);
    S.ssum = S.scnt + n_seg;
    S.hdr = p.hdr;
    S.res_dev = p.res_dev;
    S.s_lo = 0;
    S.s_hi = n_seg;
    S.final_launch = 1;
    S.chunk_total = nullptr;
    S.base_in = nullptr;
    S.base_out = nullptr;
    sl.grid_a_cap = static_cast<unsigned>(static_cast<long long>(per_sm_a) * sms);
    sl.grid_b_cap = static_cast<unsigned>(ctas);
    if (prepare_workspace(ws, need, (4ull << 56) | static_cast<unsigned long long>(n_seg), s) != cudaSuccess)
        return MVB_ERR_CUDA;
    return 0;
}

template <bool Delta>
int seg_launch_pair(SegLaunch& sl, long long s_lo, long long s_hi, bool final_launch,
                    volatile unsigned long long* chunk_total, const unsigned long long* base_in,
                    unsigned long long* base_out, cudaStream_t s) {
    constexpr int kSmemB = mvbk::kLaneSmem;
    mvbk::SegParams S = sl.S;
    S.s_lo = s_lo;
    S.s_hi = s_hi;
    S.final_launch = final_launch ? 1 : 0;
    S.chunk_total = chunk_total;
    S.base_in = base_in;
    S.base_out = base_out;
    const long long n = s_hi - s_lo;
    const long long ga = (n + mvbk::kSegWarps - 1) / mvbk::kSegWarps;  // at least one segment per warp
    // kernel A: balanced runs of at least MVB_A_ITS iterations per warp over the
    // launch's segments (clipped to the stream)
    {
        const long long its_per_seg = S.seg_bytes / mvbk::kSegASlice;
        const long long qlen = S.mis + S.len;
        const long long it0 = s_lo * its_per_seg;
        long long it1 = s_hi * its_per_seg;
        const long long it_stream = (qlen + mvbk::kSegASlice - 1) / mvbk::kSegASlice;
        if (it1 > it_stream) it1 = it_stream;
        const long long n_it = it1 > it0 ? it1 - it0 : 0;
        long long wa = (n_it + MVB_A_ITS - 1) / MVB_A_ITS;
        const long long wa_cap = static_cast<long long>(sl.grid_a_cap) * mvbk::kSegWarps;
        if (wa > wa_cap) wa = wa_cap;
        if (wa < 1) wa = 1;
        wa = (wa + mvbk::kSegWarps - 1) / mvbk::kSegWarps * mvbk::kSegWarps;
        S.a_it0 = it0;
        S.a_q = n_it / wa;
        S.a_r = n_it % wa;
        sl.grid_a_launch = static_cast<unsigned>(wa / mvbk::kSegWarps);
    }
    const unsigned grid_a = sl.grid_a_launch;
#if MVB_A_PDL
    if (Delta) {
        // programmatic dependent of whatever precedes it: only a previous decode's
        // kernel B triggers early, and A waits for it before its first write
        // (delta only: plain decodes measured 2-4% slower with it)
        cudaLaunchConfig_t ca = {};
        ca.gridDim = dim3(grid_a);
        ca.blockDim = dim3(mvbk::kSegThreads);
        ca.dynamicSmemBytes = mvbk::kASmem;
        ca.stream = s;
        cudaLaunchAttribute aa[1];
        aa[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        aa[0].val.programmaticStreamSerializationAllowed = 1;
        ca.attrs = aa;
        ca.numAttrs = 1;
        if (cudaLaunchKernelEx(&ca, mvbk::vbyte_seg_totals<Delta>, S) != cudaSuccess) return MVB_ERR_CUDA;
    } else {
        mvbk::vbyte_seg_totals<Delta><<<grid_a, mvbk::kSegThreads, mvbk::kASmem, s>>>(S);
    }
#else
    mvbk::vbyte_seg_totals<Delta><<<grid_a, mvbk::kSegThreads, mvbk::kASmem, s>>>(S);
#endif
    const unsigned grid_b = static_cast<unsigned>(ga < sl.grid_b_cap ? ga : sl.grid_b_cap);
    // programmatic dependent launch: B's CTAs launch as A's retire and wait for A's
    // results in griddepcontrol.wait (hides B's launch latency behind A's tail)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid_b);
    cfg.blockDim = dim3(mvbk::kSegThreads);
    cfg.dynamicSmemBytes = kSmemB;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, mvbk::vbyte_seg_decode<Delta>, S) != cudaSuccess) return MVB_ERR_CUDA;
    return cudaGetLastError() == cudaSuccess ? 0 : MVB_ERR_CUDA;
}

template <bool Delta>
int launch_seg(const Params& p, void* ws, size_t ws_bytes, cudaStream_t s) {
    SegLaunch sl;
    const int rc = seg_setup<Delta>(p, ws, ws_bytes, p.mis + p.len, s, sl);
    if (rc) return rc;
    return seg_launch_pair<Delta>(sl, 0, sl.S.n_seg, true, nullptr, nullptr, nullptr, s);
}

// Single-read strict decode (decode_fused.cuh): one persistent launch over
// units of mvbk::kUnit bytes.
int g_fused_swz = [] {
    const char* e = std::getenv("MVB_F_SWZ");  // (debug runs)
    return e ? std::atoi(e) : 2;
}();

struct FusedPlan {
    long long n_seg, W;
    int levels;
    long long n_at[mvbk::kFLevels];
    size_t need;
};

FusedPlan fused_plan(long long qlen, long long W_max) {
    FusedPlan f = {};
    f.n_seg = (qlen + mvbk::kUnit - 1) / mvbk::kUnit;
    f.W = std::min<long long>(W_max, (f.n_seg + mvbk::kSegWarps - 1) / mvbk::kSegWarps * mvbk::kSegWarps);
    f.levels = 1;
    long long span = 32;
    while (span <= f.n_seg && f.levels < mvbk::kFLevels) {
        span *= 32;
        ++f.levels;
    }
    f.need = kHeaderBytes;
    long long n = f.n_seg;
    for (int l = 0; l < f.levels; ++l) {
        f.n_at[l] = n;
        f.need += sizeof(mvbk::FEntry) * static_cast<size_t>(n) + (l ? 4 * static_cast<size_t>(n) : 0);
        f.need = (f.need + 15) / 16 * 16;
        n = (n + 31) / 32;
    }
    return f;
}

// extra_bytes / extra_out: room after the tree for a second kernel's arrays (the
// permissive decode's), part of the same workspace layout.
template <bool Delta, int Mode>
int launch_fused_m(const Params& p, void* ws, size_t ws_bytes, cudaStream_t s, unsigned long long* rec,
                   size_t extra_bytes = 0, char** extra_out = nullptr) {
    constexpr int mode = Mode;
    int sms = 0;
    const int per_sm = occupancy(reinterpret_cast<const void*>(mvbk::vbyte_fused_decode<Delta, Mode>), mvbk::kSegThreads,
                                 mvbk::kFSmem, &sms);
    if (per_sm < 0) return MVB_ERR_CUDA;
    const long long W_max = static_cast<long long>(per_sm) * sms * mvbk::kSegWarps;
    const FusedPlan f = fused_plan(p.mis + p.len, W_max);
    if (ws_bytes < f.need + extra_bytes) return MVB_ERR_WORKSPACE;
    if (extra_out) *extra_out = static_cast<char*>(ws) + f.need;
    mvbk::FusedParams F = {};
    mvbk::SegParams& S = F.S;
    S.in = p.in;
    S.mis = p.mis;
    S.len = p.len;
    S.count = p.count;
    S.out = p.out;
    S.prev = p.prev;
    S.prev_dev = p.prev_dev;
    S.seg_bytes = mvbk::kUnit;
    S.n_seg = f.n_seg;
    S.hdr = p.hdr;
    S.res_dev = p.res_dev;
    F.swz = g_fused_swz;
    F.narrow = (p.mis + p.len) < (1ll << 32) ? 1 : 0;
    F.mode = mode;
    F.rec = rec;
    F.levels = f.levels;
    char* b = static_cast<char*>(ws) + kHeaderBytes;
    for (int l = 0; l < f.levels; ++l) {
        F.n_at[l] = f.n_at[l];
        F.tree[l] = reinterpret_cast<mvbk::FEntry*>(b);
        b += sizeof(mvbk::FEntry) * static_cast<size_t>(f.n_at[l]);
        F.arrive[l] = l ? reinterpret_cast<unsigned*>(b) : nullptr;
        b += l ? 4 * static_cast<size_t>(f.n_at[l]) : 0;
        b = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(b) + 15) & ~static_cast<uintptr_t>(15));
    }
    const unsigned long long layout = ((extra_bytes ? 7ull : 6ull) << 56) ^ static_cast<unsigned long long>(f.n_seg);
    if (prepare_workspace(ws, f.need + extra_bytes, layout, s) != cudaSuccess) return MVB_ERR_CUDA;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(f.W / mvbk::kSegWarps));
    cfg.blockDim = dim3(mvbk::kSegThreads);
    cfg.dynamicSmemBytes = mvbk::kFSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // streams of long integers (asked for at 2.5+ bytes per integer, delta; 4+,
    // plain): the instantiation whose units of equally long 4-5-byte integers
    // take the per-integer gather and whose other delta units with such integers
    // take checked dp2a slices
    if constexpr (Mode == 0) {
        const bool st0 = MVB_F_STATIC0 > 0 && f.n_seg < MVB_F_STATIC0 * f.W;
        if (Delta ? 2 * p.len >= 5 * static_cast<long long>(p.count) : p.len >= 4 * static_cast<long long>(p.count)) {
            const void* fn = st0 ? reinterpret_cast<const void*>(mvbk::vbyte_fused_decode<Delta, 0, true, true>)
                                 : reinterpret_cast<const void*>(mvbk::vbyte_fused_decode<Delta, 0, false, true>);
            int sms2 = 0;
            if (occupancy(fn, mvbk::kSegThreads, mvbk::kFSmem, &sms2) >= per_sm) {
                const cudaError_t e = st0 ? cudaLaunchKernelEx(&cfg, mvbk::vbyte_fused_decode<Delta, 0, true, true>, F)
                                          : cudaLaunchKernelEx(&cfg, mvbk::vbyte_fused_decode<Delta, 0, false, true>, F);
                if (e != cudaSuccess) return MVB_ERR_CUDA;
                return cudaGetLastError() == cudaSuccess ? 0 : MVB_ERR_CUDA;
            }
        }
        // streams of few units per warp: the instantiation whose first round of units
        // is handed out without tickets (same registers and shared memory: the grid
        // above fits it)
        if (st0) {
            int sms2 = 0;
            const int per_sm2 = occupancy(reinterpret_cast<const void*>(mvbk::vbyte_fused_decode<Delta, 0, true>),
                                          mvbk::kSegThreads, mvbk::kFSmem, &sms2);
            if (per_sm2 >= per_sm) {
                if (cudaLaunchKernelEx(&cfg, mvbk::vbyte_fused_decode<Delta, 0, true>, F) != cudaSuccess)
                    return MVB_ERR_CUDA;
                return cudaGetLastError() == cudaSuccess ? 0 : MVB_ERR_CUDA;
            }
        }
    }
    if (cudaLaunchKernelEx(&cfg, mvbk::vbyte_fused_decode<Delta, Mode>, F) != cudaSuccess) return MVB_ERR_CUDA;
    return cudaGetLastError() == cudaSuccess ? 0 : MVB_ERR_CUDA;
}

template <bool Delta>
int launch_fused(const Params& p, void* ws, size_t ws_bytes, cudaStream_t s, int mode = 0,
                 unsigned long long* rec = nullptr, size_t extra_bytes = 0, char** extra_out = nullptr) {
    if (mode == 1) return launch_fused_m<true, 1>(p, ws, ws_bytes, s, rec);
    if (mode == 2) return launch_fused_m<true, 2>(p, ws, ws_bytes, s, rec);
    return launch_fused_m<Delta, 0>(p, ws, ws_bytes, s, rec, extra_bytes, extra_out);
}

int decode_device(const uint8_t* in, size_t in_len, size_t count, bool delta, uint32_t prev,
                  uint32_t* out, int mode, mvb_result* res_dev, void* ws, size_t ws_bytes,
                  cudaStream_t stream, const uint32_t* prev_dev = nullptr) {
    if ((in == nullptr && in_len > 0) || (out == nullptr && count > 0)) return MVB_ERR_INVALID_ARG;
    if (mode != MVB_STRICT && mode != MVB_PERMISSIVE) return MVB_ERR_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(out) & 3u) return MVB_ERR_INVALID_ARG;
    if (count == 0 || in_len == 0) {
        // decode_test.cpp:204-206 (empty request) / internal.hpp:23 (no input)
        if (res_dev) {
            mvbk::set_result_kernel<<<1, 1, 0, stream>>>(res_dev, count == 0 ? MVB_OK : MVB_TRUNCATED, 0, 0);
            if (cudaGetLastError() != cudaSuccess) return MVB_ERR_CUDA;
        }
        return 0;
    }
    const size_t mis = reinterpret_cast<uintptr_t>(in) & 15u;
    const size_t scan = scan_length(in_len, count);
    const size_t tiles = tiles_for(mis, scan);
    if (scan >= (1ull << 40)) return MVB_ERR_INVALID_ARG;
    if (ws == nullptr || ws_bytes < kHeaderBytes) return MVB_ERR_WORKSPACE;

    Params p;
    p.in = in;
    p.mis = static_cast<long long>(mis);
    p.len = static_cast<long long>(scan);
    p.count = count;
    p.out = out;
    p.prev = prev;
    p.prev_dev = prev_dev;
    p.n_tiles = static_cast<unsigned>(tiles);
    p.hdr = static_cast<WsHeader*>(ws);
    p.res_dev = res_dev;
    p.trace = nullptr;

    if (mode == MVB_STRICT && g_kernel_choice == 0)
        return delta ? launch_fused<true>(p, ws, ws_bytes, stream) : launch_fused<false>(p, ws, ws_bytes, stream);
    if (mode == MVB_STRICT && g_kernel_choice == 6)
        return delta ? launch_seg<true>(p, ws, ws_bytes, stream) : launch_seg<false>(p, ws, ws_bytes, stream);
    // per-tile kernel: permissive mode (and strict choice 1)
    p.only_if_malformed = 0;
    char* arrays = static_cast<char*>(ws) + kHeaderBytes;
    if (mode == MVB_PERMISSIVE && g_kernel_choice == 0) {
        // A stream without a malformed integer decodes alike in both modes
        // (internal.hpp:35-36 is the only difference): the strict single-read
        // decoder runs first, and the permissive kernel -- three to five times
        // slower -- only if that pass reported one (its CTAs check the result the
        // strict pass left in the header and return otherwise).  The two kernels'
        // arrays sit side by side in the workspace.
        const size_t extra = ws_need(tiles) - kHeaderBytes;
        const int rc = delta ? launch_fused<true>(p, ws, ws_bytes, stream, 0, nullptr, extra, &arrays)
                             : launch_fused<false>(p, ws, ws_bytes, stream, 0, nullptr, extra, &arrays);
        if (rc) return rc;
        p.only_if_malformed = 1;
        p.dcnt = reinterpret_cast<unsigned long long*>(arrays);
        p.dsum = p.dcnt + tiles;
        p.dmax = p.dsum + tiles;
        p.n_groups = static_cast<unsigned>(groups_for(tiles));
        p.gcnt = p.dmax + tiles;
        p.gsum = p.gcnt + p.n_groups;
        p.gacc_cnt = p.gsum + p.n_groups;
        p.gacc_sum = p.gacc_cnt + p.n_groups;
        const cudaError_t e = delta ? launch<true, mvbk::MODE_PERMISSIVE>(p, stream)
                                    : launch<false, mvbk::MODE_PERMISSIVE>(p, stream);
        return e == cudaSuccess ? 0 : MVB_ERR_CUDA;
    }
    const size_t need = ws_need(tiles);
    if (ws_bytes < need) return MVB_ERR_WORKSPACE;
    p.dcnt = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + kHeaderBytes);
    p.dsum = p.dcnt + tiles;
    p.dmax = p.dsum + tiles;
    p.n_groups = static_cast<unsigned>(groups_for(tiles));
    p.gcnt = p.dmax + tiles;
    p.gsum = p.gcnt + p.n_groups;
    p.gacc_cnt = p.gsum + p.n_groups;
    p.gacc_sum = p.gacc_cnt + p.n_groups;
    if (prepare_workspace(ws, need, (1ull << 56) | tiles, stream) != cudaSuccess) return MVB_ERR_CUDA;
    cudaError_t e;
    if (delta)
        e = mode == MVB_STRICT ? launch<true, mvbk::MODE_STRICT>(p, stream)
                               : launch<true, mvbk::MODE_PERMISSIVE>(p, stream);
    else
        e = mode == MVB_STRICT ? launch<false, mvbk::MODE_STRICT>(p, stream)
                               : launch<false, mvbk::MODE_PERMISSIVE>(p, stream);
    return e == cudaSuccess ? 0 : MVB_ERR_CUDA;
}

// Totals pass / decode pass of the single-read decoder (sharded delta decode:
// a shard's gap sum is needed by the shards after it before they decode).
int delta_totals_device(const uint8_t* in, size_t in_len, unsigned long long* rec_dev, void* ws, size_t ws_bytes,
                        cudaStream_t stream) {
    if ((in == nullptr && in_len > 0) || rec_dev == nullptr) return MVB_ERR_INVALID_ARG;
    if (in_len == 0) return cudaMemsetAsync(rec_dev, 0, 16, stream) == cudaSuccess ? 0 : MVB_ERR_CUDA;
    if (in_len >= (1ull << 40)) return MVB_ERR_INVALID_ARG;
    if (ws == nullptr || ws_bytes < kHeaderBytes) return MVB_ERR_WORKSPACE;
    Params p = {};
    p.in = in;
    p.mis = static_cast<long long>(reinterpret_cast<uintptr_t>(in) & 15u);
    p.len = static_cast<long long>(in_len);
    p.count = in_len;
    p.hdr = static_cast<WsHeader*>(ws);
    return launch_fused<true>(p, ws, ws_bytes, stream, 1, rec_dev);
}

int delta_totaled_device(const uint8_t* in, size_t in_len, size_t count, uint32_t prev, const uint32_t* prev_dev,
                         uint32_t* out, mvb_result* res_dev, void* ws, size_t ws_bytes, cudaStream_t stream) {
    if ((in == nullptr && in_len > 0) || (out == nullptr && count > 0)) return MVB_ERR_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(out) & 3u) return MVB_ERR_INVALID_ARG;
    if (count == 0 || in_len == 0) {
        if (res_dev) {
            mvbk::set_result_kernel<<<1, 1, 0, stream>>>(res_dev, count == 0 ? MVB_OK : MVB_TRUNCATED, 0, 0);
            if (cudaGetLastError() != cudaSuccess) return MVB_ERR_CUDA;
        }
        return 0;
    }
    if (ws == nullptr || ws_bytes < kHeaderBytes) return MVB_ERR_WORKSPACE;
    Params p = {};
    p.in = in;
    p.mis = static_cast<long long>(reinterpret_cast<uintptr_t>(in) & 15u);
    p.len = static_cast<long long>(in_len);  // (the totals pass covered all of in)
    p.count = count;
    p.out = out;
    p.prev = prev;
    p.prev_dev = prev_dev;
    p.hdr = static_cast<WsHeader*>(ws);
    p.res_dev = res_dev;
    return launch_fused<true>(p, ws, ws_bytes, stream, 2, nullptr);
}

// Device buffers behind the synchronous host drop-ins, cached per thread.
struct HostCtx {
    cudaStream_t stream = nullptr;  // kernels
    cudaStream_t h2d = nullptr, d2h = nullptr;  // pipelined decode: copies in each direction
    uint8_t* d_in = nullptr;
    size_t in_cap = 0;
    uint32_t* d_out = nullptr;
    size_t out_cap = 0;
    void* d_ws = nullptr;
    size_t ws_cap = 0;
    mvb_result* d_res = nullptr;
    unsigned long long* d_base = nullptr;  // pipelined decode: [count, sum] before each chunk
    // batched host decode: offsets, prevs and per-list results on the device
    unsigned long long* d_bo = nullptr;
    size_t bo_cap = 0;
    unsigned long long* d_io = nullptr;
    size_t io_cap = 0;
    uint32_t* d_prev = nullptr;
    size_t prev_cap = 0;
    mvb_result* d_lres = nullptr;
    size_t lres_cap = 0;
    // pinned, device-mapped: per-chunk integer totals and the DecodeResult the
    // final kernel writes (read by the host once the kernel's event completed)
    unsigned long long* h_tot = nullptr;
    unsigned long long* dm_tot = nullptr;
    mvb_result* h_res = nullptr;
    mvb_result* dm_res = nullptr;
    cudaEvent_t ev_in[64] = {}, ev_kst[64] = {}, ev_dec[64] = {}, ev_out[64] = {}, ev_start = nullptr;
    int last_chunks = 0;  // chunks of the last pipelined call (mvbx_host_timeline)
    bool ok = false;

    bool init() {
        if (ok) return true;
        if (cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking) != cudaSuccess)
            return false;
        if (cudaMalloc(&d_res, sizeof(mvb_result)) != cudaSuccess) return false;
        if (cudaMalloc(&d_base, 2 * 65 * sizeof(unsigned long long)) != cudaSuccess) return false;
        if (cudaHostAlloc(reinterpret_cast<void**>(&h_tot), 64 * sizeof(unsigned long long), cudaHostAllocMapped) !=
                cudaSuccess ||
            cudaHostGetDevicePointer(reinterpret_cast<void**>(&dm_tot), h_tot, 0) != cudaSuccess)
            return false;
        if (cudaHostAlloc(reinterpret_cast<void**>(&h_res), sizeof(mvb_result), cudaHostAllocMapped) != cudaSuccess ||
            cudaHostGetDevicePointer(reinterpret_cast<void**>(&dm_res), h_res, 0) != cudaSuccess)
            return false;
        for (int i = 0; i < 64; ++i)
            if (cudaEventCreate(&ev_in[i]) != cudaSuccess || cudaEventCreate(&ev_dec[i]) != cudaSuccess ||
                cudaEventCreate(&ev_kst[i]) != cudaSuccess ||
                cudaEventCreate(&ev_out[i]) != cudaSuccess)
                return false;
        if (cudaEventCreate(&ev_start) != cudaSuccess) return false;
        ok = true;
        return true;
    }
    // (zeroed on this context's own stream and waited for: the decode kernels
    // run on non-blocking streams, which the legacy default stream does not
    // order; the old buffer is freed only after this stream's earlier work)
    template <class T>
    bool grow(T*& p, size_t& cap, size_t need, bool zero) {
        if (need <= cap) return true;
        if (p) {
            if (cudaStreamSynchronize(stream) != cudaSuccess) return false;
            cudaFree(p);
        }
        p = nullptr;
        cap = 0;
        const size_t n = std::max<size_t>(need, 1u << 20);
        if (cudaMalloc(reinterpret_cast<void**>(&p), n) != cudaSuccess) return false;
        if (zero && (cudaMemsetAsync(p, 0, n, stream) != cudaSuccess || cudaStreamSynchronize(stream) != cudaSuccess))
            return false;
        cap = n;
        return true;
    }
    // per-thread buffers go with the thread (errors ignored: at process exit
    // the CUDA context may already be gone)
    ~HostCtx() {
        if (!ok) return;
        cudaStreamSynchronize(stream);
        cudaStreamSynchronize(d2h);
        for (void* q : {static_cast<void*>(d_in), static_cast<void*>(d_out), d_ws, static_cast<void*>(d_res),
                        static_cast<void*>(d_base), static_cast<void*>(d_bo), static_cast<void*>(d_io),
                        static_cast<void*>(d_prev), static_cast<void*>(d_lres)})
            if (q) cudaFree(q);
        if (h_tot) cudaFreeHost(h_tot);
        if (h_res) cudaFreeHost(h_res);
        for (int i = 0; i < 64; ++i) {
            cudaEventDestroy(ev_in[i]);
            cudaEventDestroy(ev_kst[i]);
            cudaEventDestroy(ev_dec[i]);
            cudaEventDestroy(ev_out[i]);
        }
        cudaEventDestroy(ev_start);
        cudaStreamDestroy(stream);
        cudaStreamDestroy(h2d);
        cudaStreamDestroy(d2h);
    }
};

thread_local HostCtx g_ctx;

// Pipelined host decode (strict mode, segmented kernels): the scanned bytes are
// cut into group-aligned chunks.  All H2D copies are queued on one stream;
// chunk c's kernel pair waits for its copy (it reads no byte after the chunk)
// and decodes the integers ending in it; once it completes, the host reads the
// integers ending before the chunk's end (published by the kernel into mapped
// memory) and queues the D2H of that output range on a third stream.  PCIe is
// full duplex, so the input of later chunks, the decode and the output of
// earlier chunks overlap: a call costs about max(H2D, D2H) instead of their sum.
size_t g_pipe_min = 4u << 20;     // scanned bytes from which the host drop-in pipelines
size_t g_pipe_chunk = 1u << 20;   // bytes of the first chunk (later ones double, up to 16 MB; at most 64)
bool g_pipe_grow = true;          // (tests: false keeps every chunk at g_pipe_chunk)

template <bool Delta>
int decode_host_pipelined(HostCtx& c, const uint8_t* in, size_t scan, size_t count, uint32_t prev, uint32_t* out,
                          mvb_result* res) {
    const NvtxRange range("mvb_decode_stream.pipelined");
    Params p = {};
    p.in = c.d_in;
    p.mis = 0;  // cudaMalloc'd: aligned
    p.len = static_cast<long long>(scan);
    p.count = count;
    p.out = c.d_out;
    p.prev = prev;
    p.prev_dev = nullptr;
    p.hdr = static_cast<WsHeader*>(c.d_ws);
    // the kernels write the chunk totals and the DecodeResult straight into
    // mapped host memory (a small D2H copy would queue behind the output copies)
    p.res_dev = c.dm_res;
    SegLaunch sl;
    int rc = seg_setup<Delta>(p, c.d_ws, c.ws_cap, static_cast<long long>(std::min(scan, g_pipe_chunk)), c.stream,
                                 sl);
    if (rc) return rc;
    // chunk k covers segments [cb[k], cb[k + 1]): whole groups, the first of about
    // g_pipe_chunk bytes, each next one larger by `growth` (up to 16 MB), so the
    // D2H queue stays fed while the pipeline fill is one small chunk; at most 64
    // chunks
    const long long seg = sl.S.seg_bytes, n_seg = sl.S.n_seg;
    long long cb[65];
    int n_chunks = 0;
    {
        // growth factor: the next chunk's input should arrive (H2D) no later than
        // this chunk's output leaves (D2H), i.e. about the output/input byte ratio
        // (both directions move ~55 GB/s), between 1 and 2
        const double growth =
            g_pipe_grow ? std::min(2.0, std::max(1.0, 0.9 * 4.0 * static_cast<double>(count) / scan)) : 1.0;
        long long grp0 = (static_cast<long long>(g_pipe_chunk) + 32 * seg - 1) / (32 * seg);
        if (grp0 < 1) grp0 = 1;
        for (;;) {  // (a larger first chunk until the schedule fits 64 chunks)
            const long long cap = std::max<long long>(grp0, (16ll << 20) / (32 * seg));
            long long grp = grp0, at = 0;
            n_chunks = 0;
            cb[0] = 0;
            while (at < n_seg && n_chunks < 64) {
                at = std::min(n_seg, at + 32 * grp);
                cb[++n_chunks] = at;
                grp = std::min<long long>(cap, std::max<long long>(grp, static_cast<long long>(grp * growth)));
            }
            if (at >= n_seg) break;
            grp0 *= 2;
        }
    }
    // host-side order keeps the API calls off the critical path: chunk 0's copy
    // and kernels first, then the other copies, then one chunk's kernels ahead
    // of each D2H the host waits for
    auto h2d = [&](int k) -> bool {
        const size_t b0 = static_cast<size_t>(cb[k] * seg);
        const size_t b1 = std::min(scan, static_cast<size_t>(cb[k + 1] * seg));
        if (b1 > b0 && cudaMemcpyAsync(c.d_in + b0, in + b0, b1 - b0, cudaMemcpyHostToDevice, c.h2d) != cudaSuccess)
            return false;
        return cudaEventRecord(c.ev_in[k], c.h2d) == cudaSuccess;
    };
    auto kernels = [&](int k) -> int {
        if (cudaStreamWaitEvent(c.stream, c.ev_in[k], 0) != cudaSuccess) return MVB_ERR_CUDA;
        if (cudaEventRecord(c.ev_kst[k], c.stream) != cudaSuccess) return MVB_ERR_CUDA;
        const int e = seg_launch_pair<Delta>(sl, cb[k], cb[k + 1], k == n_chunks - 1, c.dm_tot + k,
                                                k ? c.d_base + 2 * k : nullptr, c.d_base + 2 * (k + 1), c.stream);
        if (e) return e;
        if (k == n_chunks - 1 && k > 0) {  // segment totals are zero between decodes
            if (cudaMemsetAsync(sl.S.scnt, 0, 4 * static_cast<size_t>(n_seg), c.stream) != cudaSuccess ||
                cudaMemsetAsync(sl.S.ssum, 0, 4 * static_cast<size_t>(n_seg), c.stream) != cudaSuccess)
                return MVB_ERR_CUDA;
        }
        return cudaEventRecord(c.ev_dec[k], c.stream) == cudaSuccess ? 0 : MVB_ERR_CUDA;
    };
    if (cudaEventRecord(c.ev_start, c.h2d) != cudaSuccess) return MVB_ERR_CUDA;
    c.last_chunks = n_chunks;
    if (!h2d(0)) return MVB_ERR_CUDA;
    if ((rc = kernels(0)) != 0) return rc;
    for (int k = 1; k < n_chunks; ++k)
        if (!h2d(k)) return MVB_ERR_CUDA;
    size_t done = 0;
    mvb_result r = {};
    for (int k = 0; k < n_chunks; ++k) {
        if (k + 1 < n_chunks && (rc = kernels(k + 1)) != 0) return rc;
        if (cudaEventSynchronize(c.ev_dec[k]) != cudaSuccess) return MVB_ERR_CUDA;
        size_t upto;
        if (k < n_chunks - 1) {
            const unsigned long long t = static_cast<volatile unsigned long long*>(c.h_tot)[k];
            upto = static_cast<size_t>(t < count ? t : count);
        } else {
            r = *const_cast<const mvb_result*>(static_cast<volatile mvb_result*>(c.h_res));
            upto = std::max(done, static_cast<size_t>(r.values_written));
        }
        if (upto > done && cudaMemcpyAsync(out + done, c.d_out + done, (upto - done) * 4, cudaMemcpyDeviceToHost,
                                           c.d2h) != cudaSuccess)
            return MVB_ERR_CUDA;
        done = upto > done ? upto : done;
        if (cudaEventRecord(c.ev_out[k], c.d2h) != cudaSuccess) return MVB_ERR_CUDA;
    }
    if (cudaStreamSynchronize(c.d2h) != cudaSuccess) return MVB_ERR_CUDA;
    if (res) *res = r;
    return r.status;
}

int decode_host(const uint8_t* in, size_t in_len, size_t count, bool delta, uint32_t prev, uint32_t* out,
                int mode, mvb_result* res) {
    if ((in == nullptr && in_len > 0) || (out == nullptr && count > 0)) return MVB_ERR_INVALID_ARG;
    if (mode != MVB_STRICT && mode != MVB_PERMISSIVE) return MVB_ERR_INVALID_ARG;
    HostCtx& c = g_ctx;
    if (!c.init()) return MVB_ERR_CUDA;
    const size_t scan = scan_length(in_len, count);
    // at most one integer per input byte can be decoded
    const size_t n_out = std::min(count, scan);
    // the pipelined decode's segments can be finer than the one-shot decode's
    const size_t wsb = mvb_workspace_bytes(scan);
    if (!c.grow(c.d_in, c.in_cap, scan, false) || !c.grow(c.d_out, c.out_cap, n_out * 4, false) ||
        !c.grow(c.d_ws, c.ws_cap, wsb, true))
        return MVB_ERR_CUDA;
    if (mode == MVB_STRICT && count > 0 && scan >= g_pipe_min)
        return delta ? decode_host_pipelined<true>(c, in, scan, count, prev, out, res)
                     : decode_host_pipelined<false>(c, in, scan, count, prev, out, res);
    if (scan && cudaMemcpyAsync(c.d_in, in, scan, cudaMemcpyHostToDevice, c.stream) != cudaSuccess)
        return MVB_ERR_CUDA;
    const int rc = decode_device(scan ? c.d_in : nullptr, scan, count, delta, prev, count ? c.d_out : nullptr,
                                 mode, c.d_res, c.d_ws, c.ws_cap, c.stream);
    if (rc < 0) return rc;
    // the result first, then exactly out[0 .. values_written): the rest of
    // out is never touched (the device buffer may hold an earlier call's values)
    mvb_result r;
    if (cudaMemcpyAsync(&r, c.d_res, sizeof r, cudaMemcpyDeviceToHost, c.stream) != cudaSuccess ||
        cudaStreamSynchronize(c.stream) != cudaSuccess)
        return MVB_ERR_CUDA;
    const size_t n_copy = std::min<size_t>(static_cast<size_t>(r.values_written), n_out);
    if (n_copy && (cudaMemcpyAsync(out, c.d_out, n_copy * 4, cudaMemcpyDeviceToHost, c.stream) != cudaSuccess ||
                   cudaStreamSynchronize(c.stream) != cudaSuccess))
        return MVB_ERR_CUDA;
    if (res) *res = r;
    return r.status;
}

inline size_t vb_size(uint32_t x) {
    return x < (1u << 7) ? 1 : x < (1u << 14) ? 2 : x < (1u << 21) ? 3 : x < (1u << 28) ? 4 : 5;
}

}  // namespace

extern "C" {

size_t mvb_workspace_bytes(size_t in_len) {
    const size_t a = ws_need(tiles_for(15, in_len) + 1), b = 0;
    // segmented decode with 1 KiB segments (the finest any launch uses)
    const size_t n_seg = (in_len + 15) / 1024 + 1, n_grp = n_seg / 32 + 1, n_sup = n_grp / 32 + 1;
    const size_t c = kHeaderBytes + 8 * n_seg + 16 * n_grp + 16 * n_sup;
    // fused decode (fused_plan): 1 KiB segments at the finest, a 32-ary tree
    // of 16-byte entries (+ 4-byte arrival counters above level 0)
    const size_t fs = (in_len + 15) / mvbk::kUnit + 2;
    const size_t d = kHeaderBytes + 16 * fs + 20 * (fs / 31 + 2 * mvbk::kFLevels) + 16 * mvbk::kFLevels;
    // (a permissive decode keeps the per-tile kernel's arrays after the fused tree)
    return std::max(std::max(a + d, b), c);
}

int mvb_workspace_init(void* ws, size_t ws_bytes, mvb_stream_t stream) {
    if (ws == nullptr || ws_bytes < kHeaderBytes) return MVB_ERR_WORKSPACE;
    {
        std::lock_guard<std::mutex> lk(g_ws_mu);
        g_ws_layout.erase(ws);
    }
    return cudaMemsetAsync(ws, 0, ws_bytes, stream) == cudaSuccess ? 0 : MVB_ERR_CUDA;
}

int mvb_decode_device(const uint8_t* in, size_t in_len, size_t count, uint32_t* out, int mode,
                      mvb_result* res_dev, void* ws, size_t ws_bytes, mvb_stream_t stream) {
    return decode_device(in, in_len, count, false, 0, out, mode, res_dev, ws, ws_bytes, stream);
}

int mvb_decode_delta_device(const uint8_t* in, size_t in_len, size_t count, uint32_t prev, uint32_t* out,
                            int mode, mvb_result* res_dev, void* ws, size_t ws_bytes, mvb_stream_t stream) {
    return decode_device(in, in_len, count, true, prev, out, mode, res_dev, ws, ws_bytes, stream);
}

int mvb_decode_delta_device_dprev(const uint8_t* in, size_t in_len, size_t count, const uint32_t* prev_dev,
                                  uint32_t* out, int mode, mvb_result* res_dev, void* ws, size_t ws_bytes,
                                  mvb_stream_t stream) {
    if (prev_dev == nullptr) return MVB_ERR_INVALID_ARG;
    return decode_device(in, in_len, count, true, 0, out, mode, res_dev, ws, ws_bytes, stream, prev_dev);
}

int mvb_shard_carry_device(const unsigned long long* records, int n_ranks, int rank, int record_words,
                           uint32_t prev, uint32_t* carry_dev, unsigned long long* offset_dev,
                           mvb_stream_t stream) {
    if (records == nullptr || n_ranks < 1 || rank < 0 || rank >= n_ranks || record_words < 2 ||
        (carry_dev == nullptr && offset_dev == nullptr))
        return MVB_ERR_INVALID_ARG;
    mvbk::shard_carry_kernel<<<1, 32, 0, stream>>>(records, rank, record_words, prev, carry_dev, offset_dev);
    return cudaGetLastError() == cudaSuccess ? 0 : MVB_ERR_CUDA;
}

}  // extern "C"

namespace {
template <bool Delta>
int lists_device(const uint8_t* in, size_t in_len, const unsigned long long* byte_off,
                 const unsigned long long* int_off, const uint32_t* prev, size_t n_lists, const unsigned* order,
                 uint32_t* out, int mode, mvb_result* results_dev, void* ws, size_t ws_bytes, cudaStream_t s) {
    if (n_lists == 0) return 0;
    if (byte_off == nullptr || int_off == nullptr || (in == nullptr && in_len > 0)) return MVB_ERR_INVALID_ARG;
    if (mode != MVB_STRICT) return MVB_ERR_INVALID_ARG;  // permissive lists: decode each list on its own
    if (ws == nullptr || ws_bytes < kHeaderBytes) return MVB_ERR_WORKSPACE;
    if (reinterpret_cast<uintptr_t>(out) & 3u) return MVB_ERR_INVALID_ARG;
    // delta lists: the unit-based kernel (decode_lists.cuh); plain lists (and
    // kernel choice 6, for comparisons): one range decode per list
    const bool units = Delta && g_kernel_choice != 6;
    const int kSmemB = units ? mvbk::kFSmem : mvbk::kLaneSmem;
    int sms = 0;
    const int per_sm = units ? occupancy(reinterpret_cast<const void*>(mvbk::vbyte_lists_decode_units),
                                         mvbk::kSegThreads, kSmemB, &sms)
                             : occupancy(reinterpret_cast<const void*>(mvbk::vbyte_lists_decode<Delta>),
                                         mvbk::kSegThreads, kSmemB, &sms);
    if (per_sm < 0) return MVB_ERR_CUDA;
    mvbk::ListParams L;
    const size_t mis = reinterpret_cast<uintptr_t>(in) & 15u;
    L.ab = in - mis;
    L.mis0 = static_cast<long long>(mis);
    L.in_len = static_cast<long long>(in_len);
    L.byte_off = byte_off;
    L.int_off = int_off;
    L.prev = prev;
    L.order = order;
    L.n_lists = static_cast<long long>(n_lists);
    L.out = out;
    L.results = results_dev;
    L.hdr = static_cast<WsHeader*>(ws);
    const long long warps_needed = static_cast<long long>(n_lists);
    const long long ctas = std::min<long long>(static_cast<long long>(per_sm) * sms,
                                               (warps_needed + mvbk::kSegWarps - 1) / mvbk::kSegWarps);
    if (units) mvbk::vbyte_lists_decode_units<<<static_cast<unsigned>(ctas), mvbk::kSegThreads, kSmemB, s>>>(L);
    else mvbk::vbyte_lists_decode<Delta><<<static_cast<unsigned>(ctas), mvbk::kSegThreads, kSmemB, s>>>(L);
    return cudaGetLastError() == cudaSuccess ? 0 : MVB_ERR_CUDA;
}
// Batched host decode (mvb_decode_lists / mvb_decode_delta_lists): contiguous
// sub-batches of lists, about g_pipe_chunk x 4 bytes or in_len / 16 each (at
// most 64); sub-batch b's bytes, offsets and prevs go up on the H2D stream,
// its lists kernel waits for them, and the D2H of its output range
// [int_off[l0], int_off[l1]) and results waits for the kernel -- all queued up
// front, the three streams overlap.
template <bool Delta>
int lists_host(const uint8_t* in, size_t in_len, const unsigned long long* byte_off,
               const unsigned long long* int_off, const uint32_t* prev, size_t n_lists, uint32_t* out, int mode,
               mvb_result* results) {
    const NvtxRange range("mvb_decode_lists.pipelined");
    if (n_lists == 0) return 0;
    if (byte_off == nullptr || int_off == nullptr || (in == nullptr && in_len > 0)) return MVB_ERR_INVALID_ARG;
    if (mode != MVB_STRICT) return MVB_ERR_INVALID_ARG;
    const unsigned long long n_out = int_off[n_lists];
    if (n_out > 0 && out == nullptr) return MVB_ERR_INVALID_ARG;
    HostCtx& c = g_ctx;
    if (!c.init()) return MVB_ERR_CUDA;
    if (!c.grow(c.d_in, c.in_cap, in_len, false) ||
        !c.grow(c.d_out, c.out_cap, static_cast<size_t>(n_out) * 4, false) ||
        !c.grow(c.d_ws, c.ws_cap, mvb_workspace_bytes(0), true) ||
        !c.grow(c.d_bo, c.bo_cap, (n_lists + 1) * 8, false) ||
        !c.grow(c.d_io, c.io_cap, (n_lists + 1) * 8, false) ||
        !c.grow(c.d_lres, c.lres_cap, n_lists * sizeof(mvb_result), false) ||
        (prev && !c.grow(c.d_prev, c.prev_cap, n_lists * 4, false)))
        return MVB_ERR_CUDA;
    // sub-batches [lb[b], lb[b + 1])
    size_t lb[65];
    int nb = 0;
    {
        const unsigned long long total = byte_off[n_lists] - byte_off[0];
        unsigned long long target = g_pipe_grow ? std::max<unsigned long long>(4ull * g_pipe_chunk, total / 16)
                                                : std::max<unsigned long long>(g_pipe_chunk, 1);
        if (total / target > 63) target = total / 63 + 1;
        lb[0] = 0;
        size_t l = 0;
        while (l < n_lists) {
            const unsigned long long start = byte_off[l];
            size_t e = l + 1;
            while (e < n_lists && byte_off[e] - start < target) ++e;
            if (nb == 63) e = n_lists;
            lb[++nb] = e;
            l = e;
        }
    }
    for (int b = 0; b < nb; ++b) {
        const size_t l0 = lb[b], l1 = lb[b + 1];
        const size_t b0 = static_cast<size_t>(std::min<unsigned long long>(byte_off[l0], in_len));
        const size_t b1 = static_cast<size_t>(std::min<unsigned long long>(byte_off[l1], in_len));
        if (b1 > b0 && cudaMemcpyAsync(c.d_in + b0, in + b0, b1 - b0, cudaMemcpyHostToDevice, c.h2d) != cudaSuccess)
            return MVB_ERR_CUDA;
        if (cudaMemcpyAsync(c.d_bo + l0, byte_off + l0, (l1 - l0 + 1) * 8, cudaMemcpyHostToDevice, c.h2d) != cudaSuccess ||
            cudaMemcpyAsync(c.d_io + l0, int_off + l0, (l1 - l0 + 1) * 8, cudaMemcpyHostToDevice, c.h2d) != cudaSuccess)
            return MVB_ERR_CUDA;
        if (prev && cudaMemcpyAsync(c.d_prev + l0, prev + l0, (l1 - l0) * 4, cudaMemcpyHostToDevice, c.h2d) != cudaSuccess)
            return MVB_ERR_CUDA;
        if (cudaEventRecord(c.ev_in[b], c.h2d) != cudaSuccess) return MVB_ERR_CUDA;
        if (cudaStreamWaitEvent(c.stream, c.ev_in[b], 0) != cudaSuccess) return MVB_ERR_CUDA;
        const int rc = lists_device<Delta>(c.d_in, in_len, c.d_bo + l0, c.d_io + l0, prev ? c.d_prev + l0 : nullptr,
                                           l1 - l0, nullptr, n_out ? c.d_out : nullptr, mode, c.d_lres + l0, c.d_ws,
                                           c.ws_cap, c.stream);
        if (rc) return rc;
        if (cudaEventRecord(c.ev_dec[b], c.stream) != cudaSuccess) return MVB_ERR_CUDA;
        if (cudaStreamWaitEvent(c.d2h, c.ev_dec[b], 0) != cudaSuccess) return MVB_ERR_CUDA;
        const unsigned long long o0 = int_off[l0], o1 = int_off[l1];
        if (o1 > o0 && cudaMemcpyAsync(out + o0, c.d_out + o0, static_cast<size_t>(o1 - o0) * 4, cudaMemcpyDeviceToHost,
                                       c.d2h) != cudaSuccess)
            return MVB_ERR_CUDA;
        if (results && cudaMemcpyAsync(results + l0, c.d_lres + l0, (l1 - l0) * sizeof(mvb_result),
                                       cudaMemcpyDeviceToHost, c.d2h) != cudaSuccess)
            return MVB_ERR_CUDA;
    }
    return cudaStreamSynchronize(c.d2h) == cudaSuccess && cudaStreamSynchronize(c.stream) == cudaSuccess ? 0
                                                                                                   : MVB_ERR_CUDA;
}
}  // namespace

extern "C" {

int mvb_decode_lists(const uint8_t* in, size_t in_len, const unsigned long long* byte_off,
                     const unsigned long long* int_off, size_t n_lists, uint32_t* out, int mode, mvb_result* results) {
    return lists_host<false>(in, in_len, byte_off, int_off, nullptr, n_lists, out, mode, results);
}

int mvb_decode_delta_lists(const uint8_t* in, size_t in_len, const unsigned long long* byte_off,
                           const unsigned long long* int_off, const uint32_t* prev, size_t n_lists, uint32_t* out,
                           int mode, mvb_result* results) {
    return lists_host<true>(in, in_len, byte_off, int_off, prev, n_lists, out, mode, results);
}

int mvb_decode_lists_device(const uint8_t* in, size_t in_len, const unsigned long long* byte_off,
                            const unsigned long long* int_off, size_t n_lists, const unsigned* order, uint32_t* out,
                            int mode, mvb_result* results_dev, void* ws, size_t ws_bytes, mvb_stream_t stream) {
    return lists_device<false>(in, in_len, byte_off, int_off, nullptr, n_lists, order, out, mode, results_dev, ws,
                               ws_bytes, stream);
}

int mvb_decode_delta_lists_device(const uint8_t* in, size_t in_len, const unsigned long long* byte_off,
                                  const unsigned long long* int_off, const uint32_t* prev, size_t n_lists,
                                  const unsigned* order, uint32_t* out, int mode, mvb_result* results_dev, void* ws,
                                  size_t ws_bytes, mvb_stream_t stream) {
    return lists_device<true>(in, in_len, byte_off, int_off, prev, n_lists, order, out, mode, results_dev, ws,
                              ws_bytes, stream);
}

size_t mvb_encode_workspace_bytes(size_t n) {
    return ((n + mvbk::kEncTile - 1) / mvbk::kEncTile + 1) * sizeof(unsigned long long);
}

}  // extern "C"

namespace {
template <bool Delta>
int encode_device(const uint32_t* values, size_t n, uint8_t* out, unsigned long long* len_dev,
                  unsigned long long* bad_dev, void* ws, size_t ws_bytes, cudaStream_t s) {
    if (len_dev == nullptr || (n > 0 && (values == nullptr || out == nullptr))) return MVB_ERR_INVALID_ARG;
    if (Delta && bad_dev == nullptr) return MVB_ERR_INVALID_ARG;
    if (Delta && cudaMemsetAsync(bad_dev, 0xFF, sizeof(unsigned long long), s) != cudaSuccess) return MVB_ERR_CUDA;
    if (n == 0) return cudaMemsetAsync(len_dev, 0, sizeof(unsigned long long), s) == cudaSuccess ? 0 : MVB_ERR_CUDA;
    const size_t tiles = (n + mvbk::kEncTile - 1) / mvbk::kEncTile;
    if (ws == nullptr || ws_bytes < tiles * sizeof(unsigned long long)) return MVB_ERR_WORKSPACE;
    unsigned long long* tb = static_cast<unsigned long long*>(ws);
    mvbk::vbyte_enc_sizes<Delta><<<static_cast<unsigned>(tiles), mvbk::kEncThreads, 0, s>>>(values, n, tb, bad_dev);
    mvbk::vbyte_enc_scan<<<1, 1024, 0, s>>>(tb, tiles, len_dev);
    mvbk::vbyte_enc_write<Delta><<<static_cast<unsigned>(tiles), mvbk::kEncThreads, 0, s>>>(values, n, tb, out);
    return cudaGetLastError() == cudaSuccess ? 0 : MVB_ERR_CUDA;
}
}  // namespace

extern "C" {

int mvb_encode_sequence_device(const uint32_t* values, size_t n, uint8_t* out, unsigned long long* len_dev, void* ws,
                               size_t ws_bytes, mvb_stream_t stream) {
    return encode_device<false>(values, n, out, len_dev, nullptr, ws, ws_bytes, stream);
}

int mvb_encode_deltas_device(const uint32_t* sorted_values, size_t n, uint8_t* out, unsigned long long* len_dev,
                             unsigned long long* bad_index_dev, void* ws, size_t ws_bytes, mvb_stream_t stream) {
    return encode_device<true>(sorted_values, n, out, len_dev, bad_index_dev, ws, ws_bytes, stream);
}

int mvb_decode_stream(const uint8_t* in, size_t in_len, size_t count, uint32_t* out, int mode, mvb_result* res) {
    return decode_host(in, in_len, count, false, 0, out, mode, res);
}

int mvb_decode_delta_stream(const uint8_t* in, size_t in_len, size_t count, uint32_t prev, uint32_t* out,
                            int mode, mvb_result* res) {
    return decode_host(in, in_len, count, true, prev, out, mode, res);
}

int mvb_delta_totals_device(const uint8_t* in, size_t in_len, unsigned long long* rec_dev, void* ws,
                            size_t ws_bytes, mvb_stream_t stream) {
    return delta_totals_device(in, in_len, rec_dev, ws, ws_bytes, stream);
}

int mvb_decode_delta_totaled_device(const uint8_t* in, size_t in_len, size_t count, uint32_t prev,
                                    const uint32_t* prev_dev, uint32_t* out, mvb_result* res_dev, void* ws,
                                    size_t ws_bytes, mvb_stream_t stream) {
    return delta_totaled_device(in, in_len, count, prev, prev_dev, out, res_dev, ws, ws_bytes, stream);
}

int mvb_shard_cuts(const uint8_t* in, size_t in_len, int n, unsigned long long* cuts) {
    if (n < 1 || cuts == nullptr || (in == nullptr && in_len > 0)) return MVB_ERR_INVALID_ARG;
    cuts[0] = 0;
    cuts[n] = in_len;
    for (int g = 1; g < n; ++g) {
        // the first integer start at or after the even cut (a byte whose
        // predecessor terminates an integer); a continuation run with no end
        // stays whole in the shard before
        size_t p = static_cast<size_t>((static_cast<unsigned __int128>(in_len) * g) / n);
        if (p < cuts[g - 1]) p = cuts[g - 1];
        while (p < in_len && p > 0 && in[p - 1] >= 0x80u) ++p;
        cuts[g] = p;
    }
    return 0;
}

}  // extern "C"

namespace {
// Per (device, shard slot) state of mvb_decode_delta_sharded: stream, workspace,
// the shard's totals record, its DecodeResult.
struct ShardCtx {
    int dev = -1;
    cudaStream_t stream = nullptr;
    void* ws = nullptr;
    size_t ws_cap = 0;
    unsigned long long* rec = nullptr;  // [count, sum]
    mvb_result* res = nullptr;
};
std::mutex g_shard_mu;
std::deque<ShardCtx> g_shards;  // (stable references: slots only ever grow at the end)

int shard_ctx(int slot, int dev, size_t in_len, ShardCtx*& out) {
    std::lock_guard<std::mutex> lk(g_shard_mu);
    if (static_cast<int>(g_shards.size()) <= slot) g_shards.resize(slot + 1);
    ShardCtx& c = g_shards[slot];
    if (cudaSetDevice(dev) != cudaSuccess) return MVB_ERR_CUDA;
    if (c.dev != dev) {  // (a slot moved to another device: start over)
        c = ShardCtx();
        c.dev = dev;
        if (cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaMalloc(reinterpret_cast<void**>(&c.rec), 16) != cudaSuccess ||
            cudaMalloc(reinterpret_cast<void**>(&c.res), sizeof(mvb_result)) != cudaSuccess)
            return MVB_ERR_CUDA;
    }
    const size_t need = mvb_workspace_bytes(in_len);
    if (need > c.ws_cap) {
        if (c.ws && (cudaStreamSynchronize(c.stream) != cudaSuccess || cudaFree(c.ws) != cudaSuccess)) return MVB_ERR_CUDA;
        c.ws = nullptr;
        c.ws_cap = 0;
        if (cudaMalloc(&c.ws, need) != cudaSuccess) return MVB_ERR_CUDA;
        if (mvb_workspace_init(c.ws, need, c.stream) != 0 || cudaStreamSynchronize(c.stream) != cudaSuccess)
            return MVB_ERR_CUDA;
        c.ws_cap = need;
    }
    out = &c;
    return 0;
}
}  // namespace

extern "C" {

int mvb_decode_delta_sharded(int n, const int* devices, const uint8_t* const* shard_in, const size_t* shard_len,
                             size_t count, uint32_t prev, uint32_t* const* shard_out, unsigned long long* offsets,
                             mvb_result* res) {
    if (n < 1 || devices == nullptr || shard_in == nullptr || shard_len == nullptr || shard_out == nullptr)
        return MVB_ERR_INVALID_ARG;
    int dev0 = 0;
    if (cudaGetDevice(&dev0) != cudaSuccess) return MVB_ERR_CUDA;
    std::vector<ShardCtx*> C(n);
    for (int g = 0; g < n; ++g) {
        const int rc = shard_ctx(g, devices[g], shard_len[g], C[g]);
        if (rc) return rc;
    }
    const NvtxRange whole("mvb_decode_delta_sharded");
    nvtxMarkA("mvb.sharded.totals");
    // 1. totals of every shard but the last (one read of its bytes each), on
    //    each shard's own stream and device, concurrently
    std::vector<unsigned long long> rec(2 * n, 0);
    for (int g = 0; g + 1 < n; ++g) {
        if (cudaSetDevice(devices[g]) != cudaSuccess) return MVB_ERR_CUDA;
        int rc = delta_totals_device(shard_in[g], shard_len[g], C[g]->rec, C[g]->ws, C[g]->ws_cap, C[g]->stream);
        if (rc) return rc;
        if (cudaMemcpyAsync(&rec[2 * g], C[g]->rec, 16, cudaMemcpyDeviceToHost, C[g]->stream) != cudaSuccess)
            return MVB_ERR_CUDA;
    }
    nvtxMarkA("mvb.sharded.exchange");
    // 2. the exchange: 16 bytes per shard, through the host
    for (int g = 0; g + 1 < n; ++g)
        if (cudaSetDevice(devices[g]) != cudaSuccess || cudaStreamSynchronize(C[g]->stream) != cudaSuccess)
            return MVB_ERR_CUDA;
    nvtxMarkA("mvb.sharded.decode");
    // 3. every shard decodes its part of the first `count` integers from its carry
    std::vector<unsigned long long> off(n, 0), want(n, 0), byte0(n, 0);
    uint32_t carry = prev;
    for (int g = 0; g < n; ++g) {
        if (g) {
            off[g] = off[g - 1] + rec[2 * (g - 1)];
            byte0[g] = byte0[g - 1] + shard_len[g - 1];
            carry += static_cast<uint32_t>(rec[2 * (g - 1) + 1]);
        }
        const unsigned long long room = count > off[g] ? count - off[g] : 0ull;
        want[g] = (g + 1 < n) ? std::min<unsigned long long>(room, rec[2 * g]) : room;
        if (offsets) offsets[g] = off[g];
        if (cudaSetDevice(devices[g]) != cudaSuccess) return MVB_ERR_CUDA;
        int rc;
        if (g + 1 < n)
            rc = delta_totaled_device(shard_in[g], shard_len[g], static_cast<size_t>(want[g]), carry, nullptr,
                                      shard_out[g], C[g]->res, C[g]->ws, C[g]->ws_cap, C[g]->stream);
        else
            rc = decode_device(shard_in[g], shard_len[g], static_cast<size_t>(want[g]), true, carry, shard_out[g],
                               MVB_STRICT, C[g]->res, C[g]->ws, C[g]->ws_cap, C[g]->stream);
        if (rc) return rc;
    }
    nvtxMarkA("mvb.sharded.result");
    // 4. the whole-stream DecodeResult: the first shard that is not OK decides
    std::vector<mvb_result> r(n);
    for (int g = 0; g < n; ++g) {
        if (cudaSetDevice(devices[g]) != cudaSuccess ||
            cudaMemcpyAsync(&r[g], C[g]->res, sizeof(mvb_result), cudaMemcpyDeviceToHost, C[g]->stream) != cudaSuccess ||
            cudaStreamSynchronize(C[g]->stream) != cudaSuccess)
            return MVB_ERR_CUDA;
    }
    cudaSetDevice(dev0);
    mvb_result out = {};
    out.status = MVB_TRUNCATED;
    for (int g = 0; g < n; ++g) {
        const bool last = g + 1 == n || off[g] + want[g] >= count;
        if (r[g].status != MVB_OK || last) {
            out.status = r[g].status;
            out.values_written = off[g] + r[g].values_written;
            out.bytes_consumed = byte0[g] + r[g].bytes_consumed;
            if (r[g].status == MVB_TRUNCATED && r[g].values_written == 0 && g > 0 && want[g] > 0 &&
                r[g].bytes_consumed == 0)
                out.bytes_consumed = byte0[g];  // (nothing decodable in this shard: the end of the one before)
            break;
        }
    }
    if (res) *res = out;
    return out.status;
}

size_t mvb_encoded_size(uint32_t x) { return vb_size(x); }

size_t mvb_encode_one(uint32_t x, uint8_t* out) {
    size_t n = 0;
    while (x >= 0x80) {
        out[n++] = static_cast<uint8_t>(x | 0x80);
        x >>= 7;
    }
    out[n++] = static_cast<uint8_t>(x);
    return n;
}

size_t mvb_encoded_length(const uint32_t* values, size_t n) {
    size_t total = 0;
    for (size_t i = 0; i < n; ++i) total += vb_size(values[i]);
    return total;
}

size_t mvb_encode_sequence(const uint32_t* values, size_t n, uint8_t* out) {
    size_t pos = 0;
    for (size_t i = 0; i < n; ++i) pos += mvb_encode_one(values[i], out + pos);
    return pos;
}

int mvb_encode_deltas(const uint32_t* sorted_values, size_t n, uint8_t* out, size_t* out_len, size_t* bad_index) {
    uint32_t prev = 0;
    size_t pos = 0;
    for (size_t i = 0; i < n; ++i) {
        if (sorted_values[i] < prev) {
            if (bad_index) *bad_index = i;
            return MVB_ERR_DECREASING;
        }
        pos += mvb_encode_one(sorted_values[i] - prev, out + pos);
        prev = sorted_values[i];
    }
    if (out_len) *out_len = pos;
    return 0;
}

// Internal profiling switch (not part of include/mvb_cuda.h), see g_kernel_choice.
void mvbx_set_kernel(int choice) { g_kernel_choice = choice; }
#if MVB_F_TRACE
// (timeline build) rows of 64 u64 per warp of the fused decoder's grid, zeroed by the caller
int mvbx_set_fused_trace(unsigned long long* dev_rows) {
    return cudaMemcpyToSymbol(mvbk::g_ftrace, &dev_rows, sizeof(dev_rows)) == cudaSuccess ? 0 : -1;
}
#endif

// Internal profiling entry (not part of include/mvb_cuda.h): the calling
// thread's last pipelined host decode as t[4k + {0,1,2,3}] = ms from its start
// to the end of chunk k's H2D, the start and end of its kernels and the end of
// its D2H; returns the chunk count.
int mvbx_host_timeline(float* t, int cap) {
    HostCtx& c = g_ctx;
    if (!c.ok || c.last_chunks == 0) return 0;
    const int n = c.last_chunks < cap ? c.last_chunks : cap;
    for (int k = 0; k < n; ++k) {
        cudaEventElapsedTime(&t[4 * k], c.ev_start, c.ev_in[k]);
        cudaEventElapsedTime(&t[4 * k + 1], c.ev_start, c.ev_kst[k]);
        cudaEventElapsedTime(&t[4 * k + 2], c.ev_start, c.ev_dec[k]);
        cudaEventElapsedTime(&t[4 * k + 3], c.ev_start, c.ev_out[k]);
    }
    return c.last_chunks;
}

// Internal testing switch (not part of include/mvb_cuda.h): the scanned size
// from which the host drop-ins pipeline, their first chunk's bytes, and whether
// later chunks double.
void mvbx_set_host_pipeline(size_t min_bytes, size_t chunk_bytes, int grow) {
    g_pipe_min = min_bytes;
    g_pipe_chunk = chunk_bytes ? chunk_bytes : 1;
    g_pipe_grow = grow != 0;
}

// Kernels one decode call launches in steady state (bench accounting; the
// workspace re-zeroing memset runs only when a workspace changes layout).
int mvbx_kernels_per_decode(int mode) {
    return (mode == MVB_STRICT && g_kernel_choice == 6) ? 2 : 1;
}

const char* mvb_version(void) { return "mvb_cuda 0.3 (sm_100a, single-read fused VByte decoder)"; }

}  // extern "C"
