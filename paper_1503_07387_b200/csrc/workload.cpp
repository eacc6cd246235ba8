// Synthetic posting-list / integer-stream generators for the BASELINE.json
// configs, plus a multi-threaded host encoder used to build bench inputs.
//
// These are bench/test inputs, not the decode path.  Distributions follow
// SURVEY.md §8(d); the PRNG is libstdc++'s std::mt19937 / std::mt19937_64 so
// config 1 reproduces the reference tests' mixed_values() exactly
// (/root/reference/proj/tests/decode_test.cpp:22-34).  Large configs are
// generated in 2^20-value chunks, chunk c seeded with seed_seq{seed_lo,
// seed_hi, c}, so generation parallelises and stays deterministic.
//
// The encoder produces the canonical VByte format of
// /root/reference/proj/core/src/vbyte.cpp:17-39 (low digit first, 0x80 on
// every byte but the last); canonical encodings are unique, so its output is
// byte-identical to the reference encoder's (pinned in tests/test_oracle.py).
#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

namespace {

constexpr size_t kChunk = size_t{1} << 20;

template <class F>
void parallel_chunks(size_t n, F&& f) {
    const size_t chunks = (n + kChunk - 1) / kChunk;
    unsigned threads = std::max(1u, std::thread::hardware_concurrency());
    threads = static_cast<unsigned>(std::min<size_t>(threads, std::max<size_t>(chunks, 1)));
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
            for (size_t c = t; c < chunks; c += threads) {
                const size_t lo = c * kChunk, hi = std::min(n, lo + kChunk);
                f(c, lo, hi);
            }
        });
    for (auto& th : pool) th.join();
}

std::mt19937_64 chunk_rng(uint64_t seed, size_t chunk) {
    std::seed_seq seq{static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32),
                      static_cast<uint32_t>(chunk)};
    return std::mt19937_64(seq);
}

inline size_t vbyte_len(uint32_t x) {
    return x < (1u << 7) ? 1 : x < (1u << 14) ? 2 : x < (1u << 21) ? 3 : x < (1u << 28) ? 4 : 5;
}

inline size_t put_vbyte(uint32_t x, uint8_t* p) {
    size_t n = 0;
    while (x >= 0x80) {
        p[n++] = static_cast<uint8_t>(x | 0x80);
        x >>= 7;
    }
    p[n++] = static_cast<uint8_t>(x);
    return n;
}

// Recursive clustered sampler for config 3: each level keeps half the ids in
// a randomly placed dense sub-range (10%..40% of the parent width, never
// narrower than 8 ids per slot), so most gaps are 1-byte with occasional
// multi-byte jumps between clusters.
void clustered(std::mt19937_64& rng, uint64_t lo, uint64_t hi, size_t n, std::vector<uint32_t>& out) {
    if (n == 0) return;
    const uint64_t width = hi - lo;
    if (n > 32 && width <= 16 * static_cast<uint64_t>(n)) {
        // Dense leaf: selection sampling (Knuth's algorithm S), O(width).
        size_t need = n;
        std::uniform_real_distribution<double> u(0.0, 1.0);
        for (uint64_t x = lo; x < hi && need; ++x)
            if (u(rng) * static_cast<double>(hi - x) < static_cast<double>(need)) {
                out.push_back(static_cast<uint32_t>(x));
                --need;
            }
        return;
    }
    if (n <= 32) {
        // Sparse leaf: n distinct sorted ids uniform in [lo, hi) (Floyd).
        std::vector<uint32_t> pick;
        pick.reserve(n);
        for (uint64_t j = width - n; j < width; ++j) {
            const uint64_t t = std::uniform_int_distribution<uint64_t>(0, j)(rng);
            const uint32_t v = static_cast<uint32_t>(lo + t);
            if (std::find(pick.begin(), pick.end(), v) == pick.end())
                pick.push_back(v);
            else
                pick.push_back(static_cast<uint32_t>(lo + j));
        }
        std::sort(pick.begin(), pick.end());
        out.insert(out.end(), pick.begin(), pick.end());
        return;
    }
    const size_t n1 = n / 2, n2 = n - n1;
    const uint64_t mid = lo + width / 2;
    std::uniform_real_distribution<double> frac(0.10, 0.40);
    auto sub = [&](uint64_t a, uint64_t b, size_t k) {
        const uint64_t w = b - a;
        uint64_t sw = static_cast<uint64_t>(static_cast<double>(w) * frac(rng));
        sw = std::min<uint64_t>(w, std::max<uint64_t>(sw, 8 * static_cast<uint64_t>(k)));
        const uint64_t off = std::uniform_int_distribution<uint64_t>(0, w - sw)(rng);
        clustered(rng, a + off, a + off + sw, k, out);
    };
    sub(lo, mid, n1);
    sub(mid, hi, n2);
}

}  // namespace

extern "C" {

// Config 1 / reference mixed_values(n, seed): decode_test.cpp:22-34.
void mvbw_mixed_values(uint32_t* out, size_t n, uint32_t seed) {
    std::mt19937 rng(seed);
    std::uniform_int_distribution<int> len(1, 5);
    constexpr uint32_t lo[] = {0, 0, 1u << 7, 1u << 14, 1u << 21, 1u << 28};
    constexpr uint32_t hi[] = {0, (1u << 7) - 1, (1u << 14) - 1, (1u << 21) - 1, (1u << 28) - 1,
                               4294967295u};
    for (size_t i = 0; i < n; ++i) {
        const int l = len(rng);
        out[i] = std::uniform_int_distribution<uint32_t>(lo[l], hi[l])(rng);
    }
}

// Two-bracket mixture: with probability p a value uniform in [lo2, hi2],
// otherwise uniform in [lo1, hi1].  Config 2 (p=.5, [1,127] / [128,16383]),
// config 5 sweep points (all-1B, all-5B, 1B/2B mixtures).
void mvbw_mixture(uint32_t* out, size_t n, uint64_t seed, double p, uint32_t lo1, uint32_t hi1,
                  uint32_t lo2, uint32_t hi2) {
    parallel_chunks(n, [&](size_t c, size_t a, size_t b) {
        std::mt19937_64 rng = chunk_rng(seed, c);
        std::bernoulli_distribution coin(p);
        std::uniform_int_distribution<uint32_t> d1(lo1, hi1), d2(lo2, hi2);
        for (size_t i = a; i < b; ++i) out[i] = coin(rng) ? d2(rng) : d1(rng);
    });
}

// Config 4 gaps: Bernoulli(p_big) ? U[big_lo, big_hi] : 1 + Geometric(q).
void mvbw_geometric_gaps(uint32_t* out, size_t n, uint64_t seed, double q, double p_big,
                         uint32_t big_lo, uint32_t big_hi) {
    parallel_chunks(n, [&](size_t c, size_t a, size_t b) {
        std::mt19937_64 rng = chunk_rng(seed, c);
        std::bernoulli_distribution coin(p_big);
        std::geometric_distribution<uint32_t> geo(q);
        std::uniform_int_distribution<uint32_t> big(big_lo, big_hi);
        for (size_t i = a; i < b; ++i) out[i] = coin(rng) ? big(rng) : 1 + geo(rng);
    });
}

// Config 3 list lengths: round(exp(U[ln lo, ln hi])).
void mvbw_loguniform_lengths(uint32_t* out, size_t lists, uint64_t seed, uint32_t lo, uint32_t hi) {
    std::mt19937_64 rng = chunk_rng(seed, 0);
    std::uniform_real_distribution<double> u(std::log(static_cast<double>(lo)),
                                             std::log(static_cast<double>(hi)));
    for (size_t i = 0; i < lists; ++i) {
        double v = std::round(std::exp(u(rng)));
        v = std::min<double>(std::max<double>(v, lo), hi);
        out[i] = static_cast<uint32_t>(v);
    }
}

// Config 3 ids: list i (lengths[i] ids, sorted distinct, < universe) written
// at out + offsets[i] where offsets is the exclusive scan of lengths.
void mvbw_clustered_lists(uint32_t* out, const uint32_t* lengths, const uint64_t* offsets,
                          size_t lists, uint64_t seed, uint64_t universe) {
    unsigned threads = std::max(1u, std::thread::hardware_concurrency());
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
            std::vector<uint32_t> ids;
            for (size_t i = t; i < lists; i += threads) {
                std::mt19937_64 rng = chunk_rng(seed, i + 1);
                ids.clear();
                ids.reserve(lengths[i]);
                clustered(rng, 0, universe, lengths[i], ids);
                std::copy(ids.begin(), ids.end(), out + offsets[i]);
            }
        });
    for (auto& th : pool) th.join();
}

// Exact canonical encoded length of v[0..n).
size_t mvbw_encoded_length(const uint32_t* v, size_t n) {
    const size_t chunks = (n + kChunk - 1) / kChunk;
    std::vector<size_t> part(chunks, 0);
    parallel_chunks(n, [&](size_t c, size_t a, size_t b) {
        size_t s = 0;
        for (size_t i = a; i < b; ++i) s += vbyte_len(v[i]);
        part[c] = s;
    });
    size_t total = 0;
    for (size_t s : part) total += s;
    return total;
}

// Canonical encode of v[0..n) into out (sized by mvbw_encoded_length);
// returns bytes written.  Multi-threaded: per-chunk sizes, scan, then write.
size_t mvbw_encode(const uint32_t* v, size_t n, uint8_t* out) {
    const size_t chunks = (n + kChunk - 1) / kChunk;
    std::vector<size_t> part(chunks + 1, 0);
    parallel_chunks(n, [&](size_t c, size_t a, size_t b) {
        size_t s = 0;
        for (size_t i = a; i < b; ++i) s += vbyte_len(v[i]);
        part[c + 1] = s;
    });
    for (size_t c = 0; c < chunks; ++c) part[c + 1] += part[c];
    parallel_chunks(n, [&](size_t c, size_t a, size_t b) {
        uint8_t* p = out + part[c];
        for (size_t i = a; i < b; ++i) p += put_vbyte(v[i], p);
    });
    return part[chunks];
}

// Successive differences (vbyte.cpp:76-86 without the throw): returns the
// first index where v decreases, or n when v is non-decreasing.
size_t mvbw_delta(const uint32_t* v, size_t n, uint32_t* gaps) {
    uint32_t prev = 0;
    size_t bad = n;
    for (size_t i = 0; i < n; ++i) {
        if (v[i] < prev && bad == n) bad = i;
        gaps[i] = v[i] - prev;
        prev = v[i];
    }
    return bad;
}

// Segmented successive differences for concatenated lists (each list's first
// gap is taken from 0): offsets has lists+1 entries.
void mvbw_delta_lists(const uint32_t* v, const uint64_t* offsets, size_t lists, uint32_t* gaps) {
    for (size_t i = 0; i < lists; ++i) {
        uint32_t prev = 0;
        for (uint64_t j = offsets[i]; j < offsets[i + 1]; ++j) {
            gaps[j] = v[j] - prev;
            prev = v[j];
        }
    }
}

}  // extern "C"
