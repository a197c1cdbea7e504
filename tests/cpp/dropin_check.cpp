// A C++ caller of the drop-in (include/gnnsim + libgnnsim_b200.so), as a
// reference user would write it: value-type CsrGraph / FeatureMatrix in host
// memory, gnnsim::aggregate_scheduled in fp64.
//
//   dropin_check check          cache + hub-layout correctness (exit 0 = ok)
//   dropin_check bench N E D R  timing: a shuffled power-law graph of N nodes
//                               and ~E undirected edges, D-wide features, R
//                               timed calls with the hub layout on and off
//   dropin_check config C R     timing on BASELINE config C (c1..c5): the same
//                               graph as paper_2006_06608_b200/synth.py (the
//                               gnna_gen_* samplers, same seeds and top-up
//                               rounds) and random_features(n, d, seed+1000),
//                               the reference's auto_params; R warm calls
//
// Graphs: Chung-Lu sampling with the reference's own draws (mt19937_64 +
// draw_unit / draw_index, rand.hpp) and a Fisher-Yates id shuffle, so the
// hubs are scattered over the id range (the case renumbering exists for).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "gnna.h"
#include "gnnsim/gnnsim_b200.hpp"

using namespace gnnsim;

static EdgeList power_law(std::uint32_t n, std::uint64_t pairs, std::uint64_t seed, bool shuffle) {
    std::mt19937_64 rng(seed);
    const double beta = 1.0 / (2.3 - 1.0), a = 1.0 - beta, i0 = 10.0;
    const double lo = std::pow(i0, a), hi = std::pow(n + i0, a);
    auto draw = [&] {
        const double x = std::pow(lo + draw_unit(rng) * (hi - lo), 1.0 / a) - i0;
        return static_cast<NodeId>(std::min<double>(std::max(std::floor(x), 0.0), n - 1));
    };
    EdgeList el;
    el.num_nodes = n;
    el.edges.resize(pairs);
    for (auto& e : el.edges) {
        const NodeId u = draw(), v = draw();
        e = {u, v};
    }
    if (shuffle) {
        std::vector<NodeId> perm(n);
        std::iota(perm.begin(), perm.end(), 0);
        for (NodeId i = n; i > 1; --i) std::swap(perm[i - 1], perm[draw_index(rng, i)]);
        for (auto& [u, v] : el.edges) u = perm[u], v = perm[v];
    }
    return el;
}

static double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

static bool same(const FeatureMatrix& a, const FeatureMatrix& b) {
    return a.num_nodes == b.num_nodes && a.dim == b.dim &&
           std::memcmp(a.values.data(), b.values.data(), a.values.size() * sizeof(double)) == 0;
}

static bool same(const CostReport& a, const CostReport& b) {
    return a.atomic_ops == b.atomic_ops && a.global_reads == b.global_reads && a.global_writes == b.global_writes &&
           a.global_transactions == b.global_transactions && a.shared_bytes_per_block == b.shared_bytes_per_block &&
           a.cache_hits == b.cache_hits && a.cache_accesses == b.cache_accesses;
}

#define CHECK(c)                                                         \
    do {                                                                 \
        if (!(c)) {                                                      \
            std::fprintf(stderr, "FAILED %s (line %d)\n", #c, __LINE__); \
            return 1;                                                    \
        }                                                                \
    } while (0)

static int check() {
    // x = 1M x 64 doubles (512 MB > L2): the 98k hub rows of the 48 MB window
    // draw several times their uniform share of the gathers
    CsrGraph g = to_csr(power_law(1000000, 5000000, 11, true), true);
    const FeatureMatrix x = random_features(g.num_nodes, 64, 12);
    KernelParams p;
    p.ngs = 64;
    p.dw = 32;
    p.tpb = 256;
    p.dim = 64;
    EngineOptions opt;
    opt.cache = std::nullopt;
    auto [y1, r1] = aggregate_scheduled(g, x, p, Strategy::WarpShared, DimMode::Cyclic, opt);
    const b200::CallStats s1 = b200::last_call_stats();
    CHECK(!s1.cache_hit && s1.hub_rows > 0 && s1.hub_edges > 0);
    auto [y2, r2] = aggregate_scheduled(g, x, p, Strategy::WarpShared, DimMode::Cyclic, opt);
    CHECK(b200::last_call_stats().cache_hit);
    CHECK(same(y1, y2) && same(r1, r2));
    // the reference's own acceptance rule (pipeline.cpp:119-120)
    CHECK(features_close(y1, aggregate_oracle(g, x), 1e-12));
    // without the cache and the hub layout: bit-identical output and report
    setenv("GNNSIM_CACHE", "0", 1);
    setenv("GNNSIM_HUB", "0", 1);
    auto [y3, r3] = aggregate_scheduled(g, x, p, Strategy::WarpShared, DimMode::Cyclic, opt);
    CHECK(b200::last_call_stats().hub_rows == 0 && !b200::last_call_stats().cache_hit);
    CHECK(same(y1, y3) && same(r1, r3));
    // other strategies and the cache-simulating report, hub layout on vs off
    for (Strategy st : {Strategy::NaiveAtomic, Strategy::UnitSync}) {
        EngineOptions o2;  // default: LRU cache simulation on
        auto [ya, ra] = aggregate_scheduled(g, x, p, st, DimMode::Sequential, o2);
        unsetenv("GNNSIM_CACHE");
        unsetenv("GNNSIM_HUB");
        auto [yb, rb] = aggregate_scheduled(g, x, p, st, DimMode::Sequential, o2);
        CHECK(b200::last_call_stats().hub_rows > 0);
        CHECK(same(ya, yb) && same(ra, rb));
        setenv("GNNSIM_CACHE", "0", 1);
        setenv("GNNSIM_HUB", "0", 1);
    }
    unsetenv("GNNSIM_CACHE");
    unsetenv("GNNSIM_HUB");
    // a graph edited in place is not served from the cache: swap two
    // neighbours of a long row (same sizes, different CSR order)
    std::uint32_t v = 0;
    while (g.row_ptr[v + 1] - g.row_ptr[v] < 8) ++v;
    std::swap(g.col_idx[g.row_ptr[v]], g.col_idx[g.row_ptr[v] + 5]);
    auto [y4, r4] = aggregate_scheduled(g, x, p, Strategy::WarpShared, DimMode::Cyclic, opt);
    CHECK(!b200::last_call_stats().cache_hit);
    setenv("GNNSIM_CACHE", "0", 1);
    auto [y5, r5] = aggregate_scheduled(g, x, p, Strategy::WarpShared, DimMode::Cyclic, opt);
    CHECK(same(y4, y5) && same(r4, r5));
    unsetenv("GNNSIM_CACHE");
    // a small graph (x below L2): no hub layout
    CsrGraph small = to_csr(power_law(2000, 8000, 3, true), true);
    const FeatureMatrix xs = random_features(small.num_nodes, 16, 4);
    p.dim = 16;
    p.dw = 16;
    (void)aggregate_scheduled(small, xs, p, Strategy::WarpShared, DimMode::Cyclic, opt);
    CHECK(b200::last_call_stats().hub_rows == 0);
    std::printf("dropin_check ok: hub rows %u, hub gathers %llu of %zu\n", s1.hub_rows,
                (unsigned long long)s1.hub_edges, g.col_idx.size());
    return 0;
}

static int bench(std::uint32_t n, std::uint64_t pairs, std::uint32_t dim, int reps) {
    auto t0 = std::chrono::steady_clock::now();
    const CsrGraph g = to_csr(power_law(n, pairs, 8, true), true);
    const FeatureMatrix x = random_features(n, dim, 9);
    const double gen_ms = ms_since(t0);
    KernelParams p;
    p.ngs = 4096;
    p.dw = 32;
    p.tpb = 512;
    p.dim = dim;
    EngineOptions opt;
    opt.cache = std::nullopt;  // the LRU replay is a separate cost model, not the aggregation
    std::printf("{\"n\": %u, \"nnz\": %zu, \"dim\": %u, \"generate_ms\": %.1f, \"runs\": [", n, g.col_idx.size(), dim,
                gen_ms);
    for (int hub = 1; hub >= 0; --hub) {
        if (!hub) setenv("GNNSIM_HUB", "0", 1);
        b200::clear_cache();
        std::vector<double> ms;
        b200::CallStats st{};
        for (int r = 0; r < reps + 1; ++r) {
            t0 = std::chrono::steady_clock::now();
            auto res = aggregate_scheduled(g, x, p, Strategy::WarpShared, DimMode::Cyclic, opt);
            ms.push_back(ms_since(t0));
            st = b200::last_call_stats();
        }
        std::vector<double> warm(ms.begin() + 1, ms.end());
        std::sort(warm.begin(), warm.end());
        std::printf("%s{\"hub_layout\": %s, \"hub_rows\": %u, \"hub_edges\": %llu, \"first_call_ms\": %.2f, "
                    "\"warm_call_ms_median\": %.2f}",
                    hub ? "" : ", ", hub ? "true" : "false", st.hub_rows, (unsigned long long)st.hub_edges, ms[0],
                    warm[warm.size() / 2]);
    }
    unsetenv("GNNSIM_HUB");
    std::printf("]}\n");
    return 0;
}

struct Config {
    const char* kind;
    std::uint32_t n;
    std::uint64_t nnz;
    std::uint32_t dim;
    std::uint64_t seed;
    std::uint32_t communities;
    double p_intra;
    bool shuffle;
};

// synth.py CONFIGS
static bool config_of(const std::string& name, Config& c) {
    if (name == "c1") c = {"sbm", 2708, 10556, 16, 1, 7, 0.8, false};
    else if (name == "c2") c = {"sbm", 19717, 88648, 64, 2, 3, 0.8, true};
    else if (name == "c3") c = {"chung_lu", 410236, 4878874, 16, 3, 1, 0.8, false};
    else if (name == "c4") c = {"sbm", 88784, 2093194, 64, 7, 39, 0.9, false};
    else if (name == "c5") c = {"chung_lu", 10000000, 200000000, 128, 8, 1, 0.8, false};
    else return false;
    return true;
}

static void sample(const Config& c, std::uint64_t pairs, std::uint64_t seed, EdgeList& el) {
    std::vector<std::uint32_t> e(2 * pairs);
    const gnna_status st = std::strcmp(c.kind, "sbm") == 0
                               ? gnna_gen_sbm(c.n, pairs, c.communities, c.p_intra, seed, c.shuffle, e.data())
                               : gnna_gen_chung_lu(c.n, pairs, 2.3, 10.0, seed, c.shuffle, e.data());
    if (st != GNNA_OK) throw std::runtime_error("generator");
    for (std::uint64_t i = 0; i < pairs; ++i) el.edges.emplace_back(e[2 * i], e[2 * i + 1]);
}

// synth.build_graph: sample nnz/2 pairs, top up (seed + r * 1000003) until ~nnz
static CsrGraph config_graph(const Config& c) {
    EdgeList el;
    el.num_nodes = c.n;
    sample(c, c.nnz / 2, c.seed, el);
    CsrGraph g = to_csr(el, true);
    for (int r = 1; r <= 4; ++r) {
        const std::uint64_t have = g.col_idx.size();
        if (static_cast<double>(have) >= c.nnz * 0.999) break;
        const auto extra = static_cast<std::uint64_t>((static_cast<double>(c.nnz) - have) / 2 * 1.15) + 16;
        sample(c, extra, c.seed + r * 1000003ull, el);
        g = to_csr(el, true);
    }
    return g;
}

static int config_bench(const std::string& name, int reps) {
    Config c;
    if (!config_of(name, c)) return 2;
    auto t0 = std::chrono::steady_clock::now();
    const CsrGraph g = config_graph(c);
    const FeatureMatrix x = random_features(c.n, c.dim, c.seed + 1000);
    const double gen_ms = ms_since(t0);
    const KernelParams p = auto_params(ModelInputs::from_graph(g, c.dim));  // decider.cpp, as a user would
    EngineOptions opt;
    opt.cache = std::nullopt;  // the aggregation alone (the LRU replay is its own cost model)
    std::uint64_t h = 1469598103934665603ull;
    for (const auto v : g.row_ptr) h = (h ^ v) * 1099511628211ull;
    std::vector<double> ms;
    b200::CallStats st{};
    for (int r = 0; r < reps + 1; ++r) {
        t0 = std::chrono::steady_clock::now();
        auto res = aggregate_scheduled(g, x, p, Strategy::WarpShared, DimMode::Cyclic, opt);
        ms.push_back(ms_since(t0));
        st = b200::last_call_stats();
    }
    std::vector<double> warm(ms.begin() + 1, ms.end());
    std::sort(warm.begin(), warm.end());
    std::printf("{\"config\": \"%s\", \"n\": %u, \"nnz\": %zu, \"dim\": %u, \"row_ptr_fnv\": \"%016llx\", "
                "\"params\": [%u, %u, %u], \"generate_ms\": %.1f, \"first_call_ms\": %.3f, "
                "\"warm_call_ms_median\": %.3f, \"warm_calls\": %d, \"cache_hit\": %s, \"hub_rows\": %u}\n",
                name.c_str(), c.n, g.col_idx.size(), c.dim, (unsigned long long)h, p.ngs, p.dw, p.tpb, gen_ms, ms[0],
                warm[warm.size() / 2], reps, st.cache_hit ? "true" : "false", st.hub_rows);
    return 0;
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "check";
    if (mode == "check") return check();
    if (mode == "config" && argc >= 4) return config_bench(argv[2], std::atoi(argv[3]));
    if (mode == "bench" && argc >= 6)
        return bench(std::strtoul(argv[2], nullptr, 10), std::strtoull(argv[3], nullptr, 10),
                     std::strtoul(argv[4], nullptr, 10), std::atoi(argv[5]));
    std::fprintf(stderr, "usage: dropin_check check | bench N PAIRS DIM REPS | config c1..c5 REPS\n");
    return 2;
}
