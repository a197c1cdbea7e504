// Synthetic inputs for the BASELINE configs, drawn with the reference's own
// generator family: std::mt19937_64 and the explicit-arithmetic draws of
// rand.hpp:13-21 (draw_unit = 53 random bits, draw_index = 128-bit
// multiply-shift), so the same seeds give the same graphs on any standard
// library -- for this library, for bench.py's CPU reference arm and for the
// tests.  Host code (no GPU): the edge samplers split the pairs into fixed
// chunks of 2^20, chunk c drawing from mt19937_64(seed + c * 0x9E37...),
// and run the chunks on all host threads; the output does not depend on the
// thread count.  random_features is the reference's function itself
// (pipeline.cpp:57-67): one sequential stream, row-major, U[0, 1).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <random>
#include <thread>
#include <vector>

#include "gnna.h"

namespace {

inline std::size_t draw_index(std::mt19937_64& rng, std::size_t n) {
    return static_cast<std::size_t>((static_cast<unsigned __int128>(rng()) * n) >> 64);
}
inline double draw_unit(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

constexpr std::uint64_t kChunk = 1ull << 20;
constexpr std::uint64_t kGolden = 0x9E3779B97F4A7C15ull;

// Runs f(chunk, first_pair, pair_count) over the chunks of `pairs` on all host threads.
template <class F>
void chunked(std::uint64_t pairs, F&& f) {
    const std::uint64_t chunks = (pairs + kChunk - 1) / kChunk;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned nt = static_cast<unsigned>(std::min<std::uint64_t>(hw, chunks));
    std::atomic<std::uint64_t> next{0};
    auto work = [&] {
        for (std::uint64_t c; (c = next.fetch_add(1)) < chunks;) {
            const std::uint64_t b = c * kChunk;
            f(c, b, std::min(kChunk, pairs - b));
        }
    };
    if (nt <= 1) {
        work();
        return;
    }
    std::vector<std::thread> th;
    for (unsigned i = 0; i < nt; ++i) th.emplace_back(work);
    for (auto& t : th) t.join();
}

// Fisher-Yates over [0, n) with draw_index, exactly as planted_partition's shuffle (pipeline.cpp:37-44).
std::vector<std::uint32_t> shuffled_ids(std::uint32_t n, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::vector<std::uint32_t> perm(n);
    std::iota(perm.begin(), perm.end(), 0u);
    for (std::uint32_t i = n; i > 1; --i) std::swap(perm[i - 1], perm[draw_index(rng, i)]);
    return perm;
}

}  // namespace

extern "C" {

gnna_status gnna_gen_chung_lu(uint32_t n, uint64_t pairs, double gamma, double i0, uint64_t seed, int shuffle,
                              uint32_t* out_edges) {
    if (n == 0 || !(gamma > 1.0) || !(i0 > 0.0) || (pairs && !out_edges)) return GNNA_ERR_DOMAIN;
    // endpoint weight (i + i0)^(-beta), beta = 1/(gamma-1): inverse of the continuous CDF
    const double beta = 1.0 / (gamma - 1.0), a = 1.0 - beta;
    const double lo = std::pow(i0, a), hi = std::pow(static_cast<double>(n) + i0, a);
    chunked(pairs, [&](std::uint64_t c, std::uint64_t b, std::uint64_t cnt) {
        std::mt19937_64 rng(seed + c * kGolden);
        for (std::uint64_t i = 0; i < 2 * cnt; ++i) {
            const double x = std::pow(lo + draw_unit(rng) * (hi - lo), 1.0 / a) - i0;
            const double f = std::floor(x);
            out_edges[2 * b + i] = f <= 0.0 ? 0u : (f >= n - 1.0 ? n - 1 : static_cast<uint32_t>(f));
        }
    });
    if (shuffle) {
        const auto perm = shuffled_ids(n, seed ^ kGolden);
        chunked(pairs, [&](std::uint64_t, std::uint64_t b, std::uint64_t cnt) {
            for (std::uint64_t i = 2 * b; i < 2 * (b + cnt); ++i) out_edges[i] = perm[out_edges[i]];
        });
    }
    return GNNA_OK;
}

gnna_status gnna_gen_sbm(uint32_t n, uint64_t pairs, uint32_t communities, double p_intra, uint64_t seed, int shuffle,
                         uint32_t* out_edges) {
    if (n == 0 || communities == 0 || !(p_intra >= 0.0 && p_intra <= 1.0) || (pairs && !out_edges))
        return GNNA_ERR_DOMAIN;
    // equal contiguous blocks (the last takes the remainder); an endpoint
    // stays in its source's block with probability p_intra
    const std::uint32_t size = std::max<std::uint32_t>(1, n / communities);
    chunked(pairs, [&](std::uint64_t c, std::uint64_t b, std::uint64_t cnt) {
        std::mt19937_64 rng(seed + c * kGolden);
        for (std::uint64_t i = b; i < b + cnt; ++i) {
            const auto src = static_cast<std::uint32_t>(draw_index(rng, n));
            const std::uint32_t com = std::min(src / size, communities - 1);
            const std::uint32_t base = com * size, span = com == communities - 1 ? n - base : size;
            const bool intra = draw_unit(rng) < p_intra;
            const auto dst = intra ? base + static_cast<std::uint32_t>(draw_index(rng, span))
                                   : static_cast<std::uint32_t>(draw_index(rng, n));
            out_edges[2 * i] = src;
            out_edges[2 * i + 1] = dst;
        }
    });
    if (shuffle) {
        const auto perm = shuffled_ids(n, seed ^ kGolden);
        chunked(pairs, [&](std::uint64_t, std::uint64_t b, std::uint64_t cnt) {
            for (std::uint64_t i = 2 * b; i < 2 * (b + cnt); ++i) out_edges[i] = perm[out_edges[i]];
        });
    }
    return GNNA_OK;
}

// pipeline.cpp:57-67 random_features: one mt19937_64(seed) stream, row-major
// draw_unit; the F32 form is (float) of the same doubles.
gnna_status gnna_random_features(uint32_t n, uint32_t dim, uint64_t seed, int dtype, void* out) {
    if (dim == 0) return GNNA_ERR_DOMAIN;
    if (dtype != GNNA_F32 && dtype != GNNA_F64) return GNNA_ERR_DOMAIN;
    const std::uint64_t total = static_cast<std::uint64_t>(n) * dim;
    if (total && !out) return GNNA_ERR_DOMAIN;
    std::mt19937_64 rng(seed);
    if (dtype == GNNA_F64) {
        double* o = static_cast<double*>(out);
        for (std::uint64_t i = 0; i < total; ++i) o[i] = draw_unit(rng);
    } else {
        float* o = static_cast<float*>(out);
        for (std::uint64_t i = 0; i < total; ++i) o[i] = static_cast<float>(draw_unit(rng));
    }
    return GNNA_OK;
}

}  // extern "C"
