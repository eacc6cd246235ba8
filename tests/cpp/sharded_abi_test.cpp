// sharded_abi_test.cpp -- drives the C ABI's multi-GPU entry
// (mvb_decode_delta_sharded, include/mvb_cuda.h) from C++ over W shards on
// the GPUs of this process (the same device repeated when there is one), and
// checks every value and the whole-stream DecodeResult against the CPU
// oracle's decode_delta_scalar restatement (oracle/mvb_oracle.c, test-only).
// Built by __graft_entry__.build(); run by tests/test_shard.py (-m gpu).
//
//   sharded_abi_test [n_values] [shards...]     exit 0 = all cases passed
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../../include/mvb_cuda.h"

extern "C" {
typedef struct {  // oracle/mvb_oracle.c
    int32_t status;
    int32_t pad;
    uint64_t values_written;
    uint64_t bytes_consumed;
} oracle_result;
size_t oracle_encode_sequence(const uint32_t* v, size_t n, uint8_t* out);
oracle_result oracle_decode_delta(const uint8_t* in, size_t len, size_t count, uint32_t prev, uint32_t* out, int mode);
}

static int fail(const char* what, int w, size_t count) {
    std::fprintf(stderr, "FAIL %s (shards %d, count %zu)\n", what, w, count);
    return 1;
}

static int run_case(const std::vector<uint8_t>& data, size_t count, uint32_t prev, int w, int n_dev) {
    std::vector<unsigned long long> cuts(w + 1);
    if (mvb_shard_cuts(data.data(), data.size(), w, cuts.data()) != 0) return fail("cuts", w, count);
    std::vector<int> devs(w);
    std::vector<const uint8_t*> in(w);
    std::vector<uint32_t*> out(w);
    std::vector<size_t> len(w);
    for (int g = 0; g < w; ++g) {
        devs[g] = g % n_dev;
        len[g] = cuts[g + 1] - cuts[g];
        cudaSetDevice(devs[g]);
        uint8_t* d = nullptr;
        uint32_t* o = nullptr;
        cudaMalloc(&d, len[g] ? len[g] : 1);
        cudaMalloc(&o, 4 * (len[g] ? len[g] : 1));
        if (len[g]) cudaMemcpy(d, data.data() + cuts[g], len[g], cudaMemcpyHostToDevice);
        in[g] = d;
        out[g] = o;
    }
    cudaSetDevice(0);
    std::vector<unsigned long long> off(w);
    mvb_result res;
    const int rc = mvb_decode_delta_sharded(w, devs.data(), in.data(), len.data(), count, prev, out.data(),
                                            off.data(), &res);
    std::vector<uint32_t> want(count + 16);
    const oracle_result ro = oracle_decode_delta(data.data(), data.size(), count, prev, want.data(), 0);
    int bad = 0;
    if (rc != ro.status || res.status != ro.status || res.values_written != ro.values_written ||
        res.bytes_consumed != ro.bytes_consumed) {
        std::fprintf(stderr, "result %d/%d %llu %llu vs oracle %d %llu %llu\n", rc, res.status,
                     (unsigned long long)res.values_written, (unsigned long long)res.bytes_consumed, ro.status,
                     (unsigned long long)ro.values_written, (unsigned long long)ro.bytes_consumed);
        bad = fail("DecodeResult", w, count);
    }
    for (int g = 0; g < w && !bad; ++g) {
        const size_t a = off[g];
        size_t b = g + 1 < w ? off[g + 1] : ro.values_written;
        if (b > ro.values_written) b = ro.values_written;
        if (b <= a) continue;
        std::vector<uint32_t> got(b - a);
        cudaSetDevice(devs[g]);
        cudaMemcpy(got.data(), out[g], 4 * (b - a), cudaMemcpyDeviceToHost);
        for (size_t i = 0; i < b - a; ++i)
            if (got[i] != want[a + i]) {
                std::fprintf(stderr, "shard %d value %zu: %u vs %u\n", g, a + i, got[i], want[a + i]);
                bad = fail("values", w, count);
                break;
            }
    }
    for (int g = 0; g < w; ++g) {
        cudaSetDevice(devs[g]);
        cudaFree(const_cast<uint8_t*>(in[g]));
        cudaFree(out[g]);
    }
    cudaSetDevice(0);
    return bad;
}

int main(int argc, char** argv) {
    const size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1000000;
    std::vector<int> shards;
    for (int i = 2; i < argc; ++i) shards.push_back(std::atoi(argv[i]));
    if (shards.empty()) shards = {1, 2, 3, 4, 8};
    int n_dev = 0;
    if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev < 1) {
        std::fprintf(stderr, "no CUDA device\n");
        return 2;
    }
    // gaps: mostly 1-byte, some 2..3-byte, a few 5-byte (2^28+): every unit path
    std::mt19937_64 rng(20261021);
    std::vector<uint32_t> gaps(n);
    for (auto& g : gaps) {
        const uint64_t r = rng() % 1000;
        g = r < 900 ? 1 + rng() % 127 : r < 990 ? 128 + rng() % 100000 : r < 998 ? rng() % (1u << 21) : 0x10000000u + (uint32_t)(rng() % 0xE0000000u);
    }
    std::vector<uint8_t> enc(5 * n + 16);
    enc.resize(oracle_encode_sequence(gaps.data(), n, enc.data()));
    std::vector<uint8_t> trunc(enc.begin(), enc.end() - 1);
    std::vector<uint8_t> bad = enc;
    for (size_t i = 0; i < 7; ++i) bad[enc.size() / 3 + i] = 0x80;  // a malformed run
    int fails = 0, cases = 0;
    for (int w : shards) {
        fails += run_case(enc, n, 7, w, n_dev), ++cases;
        fails += run_case(enc, n / 3 + 1, 0xFFFFFFF0u, w, n_dev), ++cases;
        fails += run_case(enc, n + 5, 1, w, n_dev), ++cases;
        fails += run_case(trunc, n, 2, w, n_dev), ++cases;
        fails += run_case(bad, n, 3, w, n_dev), ++cases;
    }
    std::printf("%d/%d sharded C-ABI cases passed on %d device(s)\n", cases - fails, cases, n_dev);
    return fails ? 1 : 0;
}
