// libgnnsim_b200.so: the gnnsim:: C++ API (include/gnnsim/gnnsim_b200.hpp)
// implemented over the C-ABI of libgnna.so (include/gnna.h).
//
// Each compute entry point uploads its value-type inputs, runs the sm_100a
// kernels through gnna_* calls on the calling thread's context, and returns
// value types, exactly as the reference's functions do on the CPU.  Argument
// validation happens first and in the reference's order with its messages
// (the tests assert exception types).  Layout metadata that is not compute —
// partition_dims, map_warps, leaders_per_node, to_edge_list, the text parser,
// the seeded generators — stays on the host, as plain C++.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <sys/mman.h>
#include <fstream>
#include <atomic>
#include <list>
#include <thread>
#include <vector>
#include <map>
#include <memory>
#include <sstream>
#include <tuple>

#include "gnna.h"
#include "gnnsim/gnnsim_b200.hpp"

namespace gnnsim {
namespace {

// ------------------------------------------------------------ context
struct Ctx {
    gnna_ctx* h = nullptr;
    int device = -1;
    ~Ctx() {
        if (h) gnna_destroy(h);
    }
};

int default_device() {
    const char* e = std::getenv("GNNSIM_DEVICE");
    return e ? std::atoi(e) : 0;
}

thread_local Ctx t_ctx;
thread_local int t_device = -1;

[[noreturn]] void rethrow(gnna_ctx* c, gnna_status st) {
    const std::string msg = c ? gnna_last_error(c) : "gnna error";
    switch (st) {
        case GNNA_ERR_DOMAIN: throw DomainError(msg);
        case GNNA_ERR_INTERNAL: throw InternalError(msg);
        default: throw std::runtime_error("gnna (CUDA): " + msg);
    }
}

gnna_ctx* ctx() {
    const int want = t_device >= 0 ? t_device : default_device();
    if (!t_ctx.h || t_ctx.device != want) {
        if (t_ctx.h) gnna_destroy(t_ctx.h);
        t_ctx.h = nullptr;
        gnna_ctx* c = nullptr;
        const gnna_status st = gnna_create(want, &c);
        if (st != GNNA_OK)
            throw std::runtime_error("libgnnsim_b200 needs a B200 (sm_100) CUDA device; gnna_create failed");
        t_ctx.h = c;
        t_ctx.device = want;
    }
    return t_ctx.h;
}

void ok(gnna_status st) {
    if (st != GNNA_OK) rethrow(t_ctx.h, st);
}

// Owning device buffer.
template <class T>
class Dev {
public:
    Dev() = default;
    explicit Dev(std::size_t count) : n_(count) { ok(gnna_device_alloc(ctx(), std::max<std::size_t>(count, 1) * sizeof(T), &p_)); }
    Dev(const T* host, std::size_t count) : Dev(count) {
        if (count) ok(gnna_copy_to_device(ctx(), p_, host, count * sizeof(T)));
    }
    explicit Dev(const std::vector<T>& v) : Dev(v.data(), v.size()) {}
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    Dev(Dev&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; }
    Dev& operator=(Dev&& o) noexcept {
        if (this != &o) {
            if (p_ && t_ctx.h) gnna_device_free(t_ctx.h, p_);
            p_ = o.p_;
            n_ = o.n_;
            o.p_ = nullptr;
        }
        return *this;
    }
    ~Dev() {
        if (p_ && t_ctx.h) gnna_device_free(t_ctx.h, p_);
    }
    T* get() const { return static_cast<T*>(p_); }
    std::vector<T> host(std::size_t count) const {
        std::vector<T> v(count);
        if (count) ok(gnna_copy_to_host(ctx(), v.data(), p_, count * sizeof(T)));
        return v;
    }
    void to(T* dst, std::size_t count) const {
        if (count) ok(gnna_copy_to_host(ctx(), dst, p_, count * sizeof(T)));
    }

private:
    void* p_ = nullptr;
    std::size_t n_ = 0;
};

struct DevCsr {
    Dev<std::uint64_t> rp;
    Dev<std::uint32_t> col;
    explicit DevCsr(const CsrGraph& g) : rp(g.row_ptr), col(g.col_idx) {
        if (g.row_ptr.size() != std::size_t(g.num_nodes) + 1)
            throw DomainError("CsrGraph: row_ptr must hold num_nodes + 1 offsets");
    }
};

std::vector<std::uint32_t> flat_edges(const EdgeList& el) {
    std::vector<std::uint32_t> e(el.edges.size() * 2);
    for (std::size_t i = 0; i < el.edges.size(); ++i) {
        e[2 * i] = el.edges[i].first;
        e[2 * i + 1] = el.edges[i].second;
    }
    return e;
}

gnna_params to_c(const KernelParams& p) { return gnna_params{p.ngs, p.dw, p.tpb, p.tpw, p.dim}; }

KernelParams from_c(const gnna_params& p) {
    KernelParams k;
    k.ngs = p.ngs;
    k.dw = p.dw;
    k.tpb = p.tpb;
    k.tpw = p.tpw;
    k.dim = p.dim;
    return k;
}

gnna_model_inputs to_c(const ModelInputs& in) {
    gnna_model_inputs c{};
    c.num_nodes = in.num_nodes;
    c.num_edges = in.num_edges;
    c.dim = in.dim;
    c.max_tpb = in.max_tpb;
    c.avg_degree = in.avg_degree;
    c.stddev_degree = in.stddev_degree;
    c.smem_per_block = in.smem_per_block;
    c.capability = in.capability;
    c.alpha = in.alpha;
    return c;
}

void decider_ok(gnna_status st, const char* what) {
    if (st == GNNA_OK) return;
    const char* msg = gnna_decider_last_error();
    throw DomainError(msg && *msg ? std::string(msg) : std::string(what) + ": argument outside the evaluator's domain");
}

void check_features(const CsrGraph& g, const FeatureMatrix& x) {
    if (x.num_nodes != g.num_nodes)
        throw DomainError("feature rows (" + std::to_string(x.num_nodes) + ") do not match graph nodes (" +
                          std::to_string(g.num_nodes) + ")");
}

// ------------------------------------------------- hub rows in L2 (fp64 API)
// The reference renumbers for locality (renumber.cpp); the drop-in must keep
// the caller's order, because the fp64 results are bitwise the reference's
// summation tree, which depends on the order.  Instead the k highest-degree
// nodes' rows are COPIED into a contiguous tail of the device feature buffer
// and the plan gathers them there (gnna_hub_remap rewrites their column
// entries to n + slot): the same values in the same order, while 31 % of a
// power-law graph's gathers (C5) hit one block pinned in L2.
constexpr std::uint64_t kHubWindow = 48ull << 20;    // the L2 set-aside of bench.py's pin_hot_rows
constexpr std::uint64_t kHubMinBytes = 128ull << 20; // inputs that fit in L2 gain nothing

bool env_off(const char* name) {
    const char* e = std::getenv(name);
    return e && std::strcmp(e, "0") == 0;
}

struct Hubs {
    std::uint32_t k = 0, dim = 0;
    std::uint64_t edges = 0;
    Dev<std::uint32_t> list, col2;
};

// Hub layout for rows of `dim` doubles, or k = 0 when the graph has no
// power-law front (the hubs must draw >= 4x their uniform share of gathers).
Hubs make_hubs(const std::uint64_t* rp, const std::uint32_t* col, std::uint32_t n, std::uint64_t nnz, std::uint32_t dim) {
    Hubs h;
    h.dim = dim;
    const std::uint64_t row = std::uint64_t(dim) * sizeof(double);
    if (env_off("GNNSIM_HUB") || n == 0 || nnz == 0 || std::uint64_t(n) * row <= kHubMinBytes) return h;
    auto k = static_cast<std::uint32_t>(std::min<std::uint64_t>(n, kHubWindow / row));
    if (const char* e = std::getenv("GNNSIM_HUB_ROWS")) k = static_cast<std::uint32_t>(std::min<std::uint64_t>(n, std::strtoull(e, nullptr, 10)));
    Dev<std::uint32_t> list(k), col2(nnz);
    std::uint64_t edges = 0;
    ok(gnna_hub_remap(ctx(), rp, col, n, k, list.get(), col2.get(), &edges));
    if (static_cast<double>(edges) < 4.0 * static_cast<double>(k) / n * static_cast<double>(nnz)) return h;
    h.k = k;
    h.edges = edges;
    h.list = std::move(list);
    h.col2 = std::move(col2);
    return h;
}

using PlanPtr = std::unique_ptr<gnna_plan, void (*)(gnna_plan*)>;

PlanPtr make_plan(const std::uint64_t* rp, const std::uint32_t* col, std::uint32_t n, const gnna_params& c, int strat) {
    gnna_plan* plan = nullptr;
    ok(gnna_plan_create(ctx(), rp, col, n, 0, n, &c, strat, &plan));
    return PlanPtr(plan, gnna_plan_destroy);
}

// The features on the device, followed by copies of the hub rows when the
// hub layout is on (rows [n, n + k)).
Dev<double> upload_features(const FeatureMatrix& x, const Hubs& hubs) {
    const std::size_t body = x.values.size();
    Dev<double> ext(body + std::size_t(hubs.k) * x.dim);
    if (body) ok(gnna_copy_to_device(ctx(), ext.get(), x.values.data(), body * sizeof(double)));
    if (hubs.k) ok(gnna_gather_rows(ctx(), GNNA_F64, ext.get(), x.dim, hubs.list.get(), hubs.k, ext.get() + body));
    return ext;
}

// y = A x (fp64) over a plan built on the hub layout's columns (or the
// caller's when it is off), with the hub rows pinned in L2 for the call.
void aggregate_with_hubs(const gnna_plan* plan, const Hubs& hubs, std::uint32_t n, std::uint32_t dim, int mode,
                         const double* ext, double* dy) {
    if (!hubs.k) {
        ok(gnna_aggregate(ctx(), plan, GNNA_F64, mode, ext, dy));
        return;
    }
    const double* tail = ext + std::size_t(n) * dim;
    std::uint64_t applied = 0;
    const std::uint64_t win = std::min<std::uint64_t>(std::uint64_t(hubs.k) * dim * sizeof(double), kHubWindow);
    ok(gnna_set_l2_window(ctx(), tail, win, 1.0, &applied));
    const gnna_status st = gnna_aggregate(ctx(), plan, GNNA_F64, mode, ext, dy);
    gnna_set_l2_window(ctx(), nullptr, 0, 0.0, nullptr);
    ok(st);
}

// A zero-filled FeatureMatrix whose storage is backed by transparent huge
// pages where the kernel allows them (madvise on the reserved, untouched
// capacity before the zero-fill): the fill then takes ~500x fewer page
// faults.  Same value and type as FeatureMatrix(n, dim).
FeatureMatrix host_features(std::uint32_t n, std::uint32_t dim) {
    FeatureMatrix y;
    const std::size_t total = std::size_t(n) * dim;
    y.values.reserve(total);
    const auto a = reinterpret_cast<std::uintptr_t>(y.values.data());
    const std::uintptr_t lo = (a + (2u << 20) - 1) & ~std::uintptr_t((2u << 20) - 1);
    const std::uintptr_t hi = (a + total * sizeof(double)) & ~std::uintptr_t((2u << 20) - 1);
    if (hi > lo) madvise(reinterpret_cast<void*>(lo), hi - lo, MADV_HUGEPAGE);
    y.values.resize(total);
    y.num_nodes = n;
    y.dim = dim;
    return y;
}

// GNNSIM_TIMING=1: per-phase wall times of aggregate_scheduled on stderr.
struct PhaseTimer {
    bool on = std::getenv("GNNSIM_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[gnnsim] %-16s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

// ------------------------------------------------------ device graph cache
// The reference rebuilds its schedule inside every aggregate_scheduled call
// (engine.cpp:213-221).  A graph seen again (same storage, same sizes, same
// fingerprint) keeps its device CSR, hub layout, plans (per ngs/dw/tpb/dim/
// strategy) and CostReports across calls.  The fingerprint hashes ALL of
// row_ptr and col_idx (64-bit multiply-xor over 8-byte words, 4 lanes, in
// 1 MiB chunks on all host threads, chunk hashes combined in order), so a
// graph edited in place anywhere is rebuilt.  GNNSIM_CACHE=0 turns the
// cache off.
std::uint64_t mix(std::uint64_t h, std::uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    return h * 0xff51afd7ed558ccdull;
}

std::uint64_t hash_bytes(const unsigned char* p, std::size_t bytes) {
    std::uint64_t l[4] = {0x243f6a8885a308d3ull, 0x13198a2e03707344ull, 0xa4093822299f31d0ull, 0x082efa98ec4e6c89ull};
    std::size_t i = 0;
    for (; i + 32 <= bytes; i += 32)
        for (int k = 0; k < 4; ++k) {
            std::uint64_t w;
            std::memcpy(&w, p + i + 8 * k, 8);
            l[k] = (l[k] ^ w) * 0x100000001b3ull;
        }
    for (; i + 8 <= bytes; i += 8) {  // the remaining whole words
        std::uint64_t w;
        std::memcpy(&w, p + i, 8);
        l[0] = (l[0] ^ w) * 0x100000001b3ull;
    }
    std::uint64_t tail = 0;  // the last < 8 bytes
    std::memcpy(&tail, p + i, bytes - i);
    return mix(mix(mix(mix(l[0], l[1]), l[2]), l[3]), tail ^ bytes);
}

std::uint64_t hash_parallel(const void* data, std::size_t bytes) {
    constexpr std::size_t kChunk = 1u << 20;
    const std::size_t chunks = (bytes + kChunk - 1) / kChunk;
    std::vector<std::uint64_t> part(chunks);
    const auto* p = static_cast<const unsigned char*>(data);
    const unsigned nt = static_cast<unsigned>(
        std::min<std::size_t>(chunks, std::max(1u, std::min(16u, std::thread::hardware_concurrency()))));
    std::atomic<std::size_t> next{0};
    auto work = [&] {
        for (std::size_t c; (c = next.fetch_add(1)) < chunks;)
            part[c] = hash_bytes(p + c * kChunk, std::min(kChunk, bytes - c * kChunk));
    };
    if (nt <= 1) {
        work();
    } else {
        std::vector<std::thread> th;
        for (unsigned i = 0; i < nt; ++i) th.emplace_back(work);
        for (auto& t : th) t.join();
    }
    std::uint64_t h = bytes;
    for (const auto v : part) h = mix(h, v);
    return h;
}

std::uint64_t fingerprint(const CsrGraph& g) {
    return mix(mix(mix(g.num_nodes, g.col_idx.size()), hash_parallel(g.row_ptr.data(), g.row_ptr.size() * 8)),
               hash_parallel(g.col_idx.data(), g.col_idx.size() * 4));
}

struct CachedGraph {
    const void* rp_data = nullptr;
    const void* col_data = nullptr;
    std::uint32_t n = 0;
    std::uint64_t nnz = 0, fp = 0;
    std::unique_ptr<DevCsr> d;
    std::unique_ptr<Hubs> hubs;
    std::map<std::tuple<std::uint32_t, std::uint32_t, std::uint32_t, std::uint32_t, int, bool>, PlanPtr> plans;
    std::map<std::tuple<std::uint32_t, std::uint32_t, std::uint32_t, std::uint32_t, int, int, std::uint64_t,
                        std::uint64_t, std::uint64_t>,
             gnna_cost>
        costs;

    const gnna_plan* plan(const gnna_params& c, int strat, bool hub) {
        const auto key = std::make_tuple(c.ngs, c.dw, c.tpb, c.dim, strat, hub);
        auto it = plans.find(key);
        if (it == plans.end())
            it = plans.emplace(key, make_plan(d->rp.get(), hub ? hubs->col2.get() : d->col.get(), n, c, strat)).first;
        return it->second.get();
    }
    const Hubs& hub_layout(std::uint32_t dim) {
        if (!hubs || hubs->dim != dim) {
            // plans over the previous layout's col2 must go with it
            for (auto it = plans.begin(); it != plans.end();) it = std::get<5>(it->first) ? plans.erase(it) : std::next(it);
            hubs = std::make_unique<Hubs>(make_hubs(d->rp.get(), d->col.get(), n, nnz, dim));
        }
        return *hubs;
    }
};

thread_local std::list<CachedGraph> t_graphs;  // most recent first
constexpr std::size_t kCachedGraphs = 4;

thread_local b200::CallStats t_stats;

CachedGraph& cached_graph(const CsrGraph& g, std::unique_ptr<CachedGraph>& scratch) {
    t_stats = b200::CallStats{};
    if (env_off("GNNSIM_CACHE")) {  // a throwaway entry per call
        scratch = std::make_unique<CachedGraph>();
        scratch->n = g.num_nodes;
        scratch->nnz = g.col_idx.size();
        scratch->d = std::make_unique<DevCsr>(g);
        return *scratch;
    }
    const std::uint64_t fp = fingerprint(g);
    for (auto it = t_graphs.begin(); it != t_graphs.end(); ++it)
        if (it->rp_data == g.row_ptr.data() && it->col_data == g.col_idx.data() && it->n == g.num_nodes &&
            it->nnz == g.col_idx.size() && it->fp == fp) {
            t_graphs.splice(t_graphs.begin(), t_graphs, it);
            t_stats.cache_hit = true;
            return t_graphs.front();
        }
    auto d = std::make_unique<DevCsr>(g);  // validates before the entry exists
    t_graphs.emplace_front();
    CachedGraph& e = t_graphs.front();
    e.rp_data = g.row_ptr.data();
    e.col_data = g.col_idx.data();
    e.n = g.num_nodes;
    e.nnz = g.col_idx.size();
    e.fp = fp;
    e.d = std::move(d);
    while (t_graphs.size() > kCachedGraphs) t_graphs.pop_back();
    return e;
}

NodeId parse_id(const std::string& tok, std::size_t line) {
    if (tok.empty()) throw ParseError("empty token", line);
    if (tok[0] == '-') throw ParseError("negative node id '" + tok + "'", line);
    std::uint64_t v = 0;
    for (char c : tok) {
        if (c < '0' || c > '9') throw ParseError("malformed token '" + tok + "'", line);
        v = v * 10 + std::uint64_t(c - '0');
        if (v > 0xFFFFFFFEull) throw ParseError("node id '" + tok + "' out of range", line);
    }
    return static_cast<NodeId>(v);
}

}  // namespace

void set_device(int device) { t_device = device; }

// =============================================================== graph
EdgeList load_edge_list(std::istream& in) {
    EdgeList el;
    std::optional<NodeId> declared;
    NodeId span = 0;  // 1 + largest id seen
    std::string text;
    for (std::size_t line = 1; std::getline(in, text); ++line) {
        std::istringstream ss(text);
        std::string a, b, rest;
        if (!(ss >> a) || a[0] == '#' || a[0] == '%') continue;
        if (a == "nodes") {
            if (!(ss >> b)) throw ParseError("header 'nodes' without a count", line);
            declared = parse_id(b, line);
            continue;
        }
        if (!(ss >> b)) throw ParseError("expected 'src dst', got one token", line);
        if (ss >> rest) throw ParseError("trailing token '" + rest + "'", line);
        const NodeId s = parse_id(a, line), d = parse_id(b, line);
        el.edges.emplace_back(s, d);
        span = std::max({span, s + 1, d + 1});
    }
    if (declared) {
        if (span > *declared)
            throw ParseError("node id " + std::to_string(span - 1) + " exceeds declared node count " +
                             std::to_string(*declared));
        el.num_nodes = *declared;
    } else {
        el.num_nodes = span;
    }
    return el;
}

EdgeList load_edge_list_file(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw IoError("cannot open '" + path + "'");
    return load_edge_list(f);
}

CsrGraph to_csr(const EdgeList& el, bool symmetrize) {
    CsrGraph g;
    g.num_nodes = el.num_nodes;
    const Dev<std::uint32_t> e(flat_edges(el));
    Dev<std::uint64_t> rp(std::size_t(el.num_nodes) + 1);
    std::uint64_t nnz = 0;
    ok(gnna_to_csr(ctx(), el.num_nodes, e.get(), el.edges.size(), symmetrize, rp.get(), nullptr, &nnz));
    Dev<std::uint32_t> col(nnz);
    ok(gnna_to_csr(ctx(), el.num_nodes, e.get(), el.edges.size(), symmetrize, rp.get(), col.get(), &nnz));
    g.row_ptr = rp.host(std::size_t(el.num_nodes) + 1);
    g.col_idx = col.host(nnz);
    return g;
}

EdgeList to_edge_list(const CsrGraph& g) {
    EdgeList el;
    el.num_nodes = g.num_nodes;
    el.edges.reserve(g.num_edges());
    for (NodeId v = 0; v < g.num_nodes; ++v)
        for (NodeId u : g.neighbors(v)) el.edges.emplace_back(v, u);
    return el;
}

DegreeStats degree_stats(const CsrGraph& g) {
    if (g.num_nodes == 0) throw DomainError("degree_stats: graph has no nodes");
    const Dev<std::uint64_t> rp(g.row_ptr);
    DegreeStats s;
    ok(gnna_degree_stats(ctx(), rp.get(), g.num_nodes, &s.avg_degree, &s.max_degree, &s.stddev_degree));
    return s;
}

double aes(const EdgeList& el) {
    if (el.edges.empty()) throw DomainError("no edges in the input");
    const Dev<std::uint32_t> e(flat_edges(el));
    double out = 0.0;
    ok(gnna_aes(ctx(), e.get(), el.edges.size(), &out));
    return out;
}

FeatureMatrix ones_features(std::uint32_t n, std::uint32_t dim) {
    if (n == 0 || dim == 0) throw DomainError("ones_features: n and dim must be >= 1");
    FeatureMatrix x(n, dim);
    std::fill(x.values.begin(), x.values.end(), 1.0);
    return x;
}

// ============================================================ schedule
void KernelParams::validate() const {
    const gnna_params c = to_c(*this);
    ok(gnna_validate_params(ctx(), &c));
}

std::vector<NeighborGroup> partition_neighbors(const CsrGraph& g, std::uint32_t ngs) {
    if (ngs < 1) throw DomainError("partition_neighbors: ngs must be >= 1");
    const Dev<std::uint64_t> rp(g.row_ptr);
    std::uint64_t G = 0;
    ok(gnna_count_groups(ctx(), rp.get(), g.num_nodes, ngs, &G));
    Dev<std::uint64_t> pp(G + 1);
    Dev<std::uint32_t> tgt(G);
    ok(gnna_partition_neighbors(ctx(), rp.get(), g.num_nodes, ngs, pp.get(), tgt.get()));
    const auto p = pp.host(G + 1);
    const auto t = tgt.host(G);
    std::vector<NeighborGroup> out(G);
    for (std::uint64_t u = 0; u < G; ++u) out[u] = NeighborGroup{std::uint32_t(u), t[u], p[u], p[u + 1]};
    return out;
}

DimAssignment partition_dims(std::uint32_t dim, std::uint32_t dw, DimMode mode) {
    if (dw < 1) throw DomainError("partition_dims: dw must be >= 1");
    DimAssignment a;
    a.mode = mode;
    a.lanes.assign(dw, {});
    const std::uint32_t chunk = (dim + dw - 1) / dw;
    for (std::uint32_t t = 0; t < dw; ++t) {
        if (mode == DimMode::Cyclic) {
            for (std::uint32_t d = t; d < dim; d += dw) a.lanes[t].push_back(d);
        } else {
            const std::uint32_t lo = t * chunk, hi = std::min(lo + chunk, dim);
            for (std::uint32_t d = lo; d < hi; ++d) a.lanes[t].push_back(d);
        }
    }
    return a;
}

WarpSchedule map_warps(std::vector<NeighborGroup> groups, const KernelParams& params) {
    params.validate();
    WarpSchedule s;
    s.warps = std::move(groups);
    s.warp_per_block = params.warps_per_block();
    return s;
}

// ============================================================= memplan
MemPlan build_mem_plan(const WarpSchedule& sched, const KernelParams& params) {
    params.validate();
    if (sched.warp_per_block == 0 || sched.warp_per_block != params.warps_per_block())
        throw DomainError("build_mem_plan: schedule block width does not match params");
    const std::size_t G = sched.warps.size();
    std::vector<std::uint32_t> targets(G);
    for (std::size_t i = 0; i < G; ++i) targets[i] = sched.warps[i].target;
    const Dev<std::uint32_t> t(targets);
    Dev<std::uint8_t> slot(G), lead(G);
    const gnna_params c = to_c(params);
    MemPlan plan;
    ok(gnna_build_mem_plan(ctx(), t.get(), G, &c, slot.get(), lead.get(), &plan.shared_bytes_per_block));
    const auto s = slot.host(G);
    const auto l = lead.host(G);
    plan.entries.resize(G);
    for (std::size_t i = 0; i < G; ++i) plan.entries[i] = WarpPlanEntry{s[i], targets[i], l[i] != 0};
    return plan;
}

std::map<NodeId, std::uint32_t> leaders_per_node(const MemPlan& plan, const WarpSchedule& sched) {
    if (plan.entries.size() != sched.warps.size()) throw DomainError("leaders_per_node: plan does not match schedule");
    std::map<NodeId, std::uint32_t> n;
    for (const auto& e : plan.entries)
        if (e.leader) ++n[e.node];
    return n;
}

// ============================================================== engine
void CacheConfig::validate() const {
    if (line_size == 0) throw DomainError("cache line size must be positive");
    if (capacity < line_size || capacity % line_size != 0)
        throw DomainError("cache capacity must be a positive multiple of the line size");
}

FeatureMatrix aggregate_oracle(const CsrGraph& g, const FeatureMatrix& x) {
    check_features(g, x);
    const DevCsr d(g);
    const Dev<double> dx(x.values);
    Dev<double> dy(x.values.size());
    ok(gnna_aggregate_rows(ctx(), GNNA_F64, d.rp.get(), d.col.get(), g.num_nodes, x.dim, dx.get(), dy.get()));
    FeatureMatrix y(g.num_nodes, x.dim);
    dy.to(y.values.data(), y.values.size());
    return y;
}

std::pair<FeatureMatrix, CostReport> aggregate_scheduled(const CsrGraph& g, const FeatureMatrix& x,
                                                         const KernelParams& params, Strategy strategy,
                                                         DimMode dim_mode, const EngineOptions& opts) {
    params.validate();
    check_features(g, x);
    if (x.dim != params.dim)
        throw DomainError("feature dim (" + std::to_string(x.dim) + ") does not match kernel dim (" +
                          std::to_string(params.dim) + ")");
    if (opts.transaction_line_bytes == 0) throw DomainError("transaction line size must be positive");
    if (opts.cache) opts.cache->validate();
    PhaseTimer pt;
    // the output's host allocation (zero-filled, first-touch page faults: the
    // largest host cost at C3 / C4) proceeds on a helper thread meanwhile
    std::unique_ptr<FeatureMatrix> yp;
    std::exception_ptr alloc_err;
    std::thread alloc([&] {
        try {
            yp = std::make_unique<FeatureMatrix>(host_features(g.num_nodes, x.dim));
        } catch (...) {
            alloc_err = std::current_exception();  // rethrown on the caller's thread after the join
        }
    });
    struct Join {
        std::thread& t;
        ~Join() {
            if (t.joinable()) t.join();
        }
    } join{alloc};
    std::unique_ptr<CachedGraph> scratch;
    CachedGraph& G = cached_graph(g, scratch);
    const Hubs& hubs = G.hub_layout(x.dim);
    t_stats.hub_rows = hubs.k;
    t_stats.hub_edges = hubs.edges;
    pt.mark("graph");
    const Dev<double> dx = upload_features(x, hubs);
    Dev<double> dy(x.values.size());
    pt.mark("upload");
    const gnna_params c = to_c(params);
    const int strat = strategy == Strategy::NaiveAtomic ? GNNA_NAIVE_ATOMIC
                      : strategy == Strategy::UnitSync  ? GNNA_UNIT_SYNC
                                                        : GNNA_WARP_SHARED;
    const int mode = dim_mode == DimMode::Sequential ? GNNA_DIM_SEQUENTIAL : GNNA_DIM_CYCLIC;
    aggregate_with_hubs(G.plan(c, strat, hubs.k > 0), hubs, g.num_nodes, x.dim, mode, dx.get(), dy.get());
    // CostReport of the reference's model: on the caller's columns (transaction
    // lines are address-dependent), cached per (params, strategy, dim mode, options)
    const std::uint64_t cap = opts.cache ? opts.cache->capacity : 0, cl = opts.cache ? opts.cache->line_size : 0;
    const auto ckey = std::make_tuple(c.ngs, c.dw, c.tpb, c.dim, strat, mode, opts.transaction_line_bytes, cap, cl);
    auto cit = G.costs.find(ckey);
    if (cit == G.costs.end()) {
        gnna_cost cost{};
        ok(gnna_cost_report(ctx(), G.plan(c, strat, false), mode, opts.transaction_line_bytes, cap, cl, &cost));
        cit = G.costs.emplace(ckey, cost).first;
    }
    const gnna_cost cost = cit->second;
    ok(gnna_synchronize(ctx()));
    pt.mark("aggregate+cost");
    alloc.join();
    if (alloc_err) std::rethrow_exception(alloc_err);
    FeatureMatrix y = std::move(*yp);
    pt.mark("alloc_y (join)");
    dy.to(y.values.data(), y.values.size());
    pt.mark("download");
    CostReport r;
    r.atomic_ops = cost.atomic_ops;
    r.global_reads = cost.global_reads;
    r.global_writes = cost.global_writes;
    r.global_transactions = cost.global_transactions;
    r.shared_bytes_per_block = cost.shared_bytes_per_block;
    r.cache_hits = cost.cache_hits;
    r.cache_accesses = cost.cache_accesses;
    return {std::move(y), r};
}

bool features_close(const FeatureMatrix& a, const FeatureMatrix& b, double rel_tol) {
    if (a.num_nodes != b.num_nodes || a.dim != b.dim) return false;
    for (std::size_t i = 0; i < a.values.size(); ++i) {
        const double p = a.values[i], q = b.values[i];
        if (std::fabs(p - q) > rel_tol * std::max(std::fabs(p), std::fabs(q))) return false;
    }
    return true;
}

std::uint64_t count_transactions(std::span<const std::uint64_t> addresses, std::uint64_t line) {
    if (line == 0) throw DomainError("transaction line size must be positive");
    std::vector<std::uint64_t> l(addresses.size());
    for (std::size_t i = 0; i < addresses.size(); ++i) l[i] = addresses[i] / line;
    std::sort(l.begin(), l.end());
    return static_cast<std::uint64_t>(std::unique(l.begin(), l.end()) - l.begin());
}

std::pair<std::uint64_t, std::uint64_t> simulate_cache(const CsrGraph& g, const WarpSchedule& sched,
                                                       const CacheConfig& cfg, std::uint32_t dim) {
    cfg.validate();
    if (dim == 0) throw DomainError("dim must be positive");
    const std::size_t G = sched.warps.size();
    std::vector<std::uint64_t> b(G), e(G);
    for (std::size_t i = 0; i < G; ++i) {
        b[i] = sched.warps[i].begin;
        e[i] = sched.warps[i].end;
    }
    const Dev<std::uint32_t> col(g.col_idx);
    const Dev<std::uint64_t> db(b), de(e);
    std::uint64_t hits = 0, acc = 0;
    ok(gnna_simulate_cache_ranges(ctx(), col.get(), db.get(), de.get(), G, sched.warp_per_block, cfg.capacity,
                                  cfg.line_size, dim, &hits, &acc));
    return {hits, acc};
}

FeatureMatrix gcn_layer(const CsrGraph& g, const FeatureMatrix& x, const FeatureMatrix& w, bool add_self_loops) {
    check_features(g, x);
    if (w.num_nodes != x.dim)
        throw DomainError("weight rows (" + std::to_string(w.num_nodes) + ") do not match input dim (" +
                          std::to_string(x.dim) + ")");
    const DevCsr d(g);
    const Dev<double> dx(x.values), dw(w.values);
    Dev<double> dy(std::size_t(g.num_nodes) * w.dim);
    ok(gnna_gcn_forward(ctx(), GNNA_F64, d.rp.get(), d.col.get(), g.num_nodes, dx.get(), x.dim, dw.get(), w.dim,
                        add_self_loops, dy.get()));
    FeatureMatrix y(g.num_nodes, w.dim);
    dy.to(y.values.data(), y.values.size());
    return y;
}

FeatureMatrix gin_layer(const CsrGraph& g, const FeatureMatrix& x, double eps, const AffineMap& mlp) {
    check_features(g, x);
    if (mlp.weight.num_nodes != x.dim)
        throw DomainError("affine weight rows (" + std::to_string(mlp.weight.num_nodes) +
                          ") do not match input dim (" + std::to_string(x.dim) + ")");
    if (mlp.bias.size() != mlp.weight.dim)
        throw DomainError("affine bias size (" + std::to_string(mlp.bias.size()) + ") does not match output dim (" +
                          std::to_string(mlp.weight.dim) + ")");
    const DevCsr d(g);
    const Dev<double> dx(x.values), dw(mlp.weight.values), db(mlp.bias);
    Dev<double> dy(std::size_t(g.num_nodes) * mlp.weight.dim);
    ok(gnna_gin_forward(ctx(), GNNA_F64, d.rp.get(), d.col.get(), g.num_nodes, dx.get(), x.dim, eps, dw.get(),
                        mlp.weight.dim, db.get(), dy.get()));
    FeatureMatrix y(g.num_nodes, mlp.weight.dim);
    dy.to(y.values.data(), y.values.size());
    return y;
}

namespace {
// Transposed CSR of g on the device (for the adjoint aggregation).
struct DevTranspose {
    Dev<std::uint64_t> rp;
    Dev<std::uint32_t> col;
    DevTranspose(const DevCsr& d, const CsrGraph& g) : rp(std::size_t(g.num_nodes) + 1), col(g.num_edges()) {
        ok(gnna_csr_transpose(ctx(), d.rp.get(), d.col.get(), g.num_nodes, rp.get(), col.get()));
    }
};
}  // namespace

GcnGrads gcn_layer_backward(const CsrGraph& g, const FeatureMatrix& x, const FeatureMatrix& w,
                            const FeatureMatrix& dy, bool add_self_loops) {
    check_features(g, x);
    if (w.num_nodes != x.dim) throw DomainError("weight rows do not match input dim");
    if (dy.num_nodes != g.num_nodes || dy.dim != w.dim) throw DomainError("dy shape does not match the layer output");
    const DevCsr d(g);
    const DevTranspose t(d, g);
    const Dev<double> dx_in(x.values), dw_in(w.values), ddy(dy.values);
    Dev<double> gx(x.values.size()), gw(w.values.size());
    ok(gnna_gcn_backward(ctx(), GNNA_F64, d.rp.get(), d.col.get(), t.rp.get(), t.col.get(), g.num_nodes, dx_in.get(),
                         x.dim, dw_in.get(), w.dim, add_self_loops, ddy.get(), gx.get(), gw.get()));
    GcnGrads r{FeatureMatrix(x.num_nodes, x.dim), FeatureMatrix(w.num_nodes, w.dim)};
    gx.to(r.dx.values.data(), r.dx.values.size());
    gw.to(r.dw.values.data(), r.dw.values.size());
    return r;
}

GinGrads gin_layer_backward(const CsrGraph& g, const FeatureMatrix& x, double eps, const AffineMap& mlp,
                            const FeatureMatrix& dy) {
    check_features(g, x);
    if (mlp.weight.num_nodes != x.dim || mlp.bias.size() != mlp.weight.dim)
        throw DomainError("affine map does not match the input dim");
    if (dy.num_nodes != g.num_nodes || dy.dim != mlp.weight.dim)
        throw DomainError("dy shape does not match the layer output");
    const DevCsr d(g);
    const DevTranspose t(d, g);
    const Dev<double> dx_in(x.values), dw_in(mlp.weight.values), db_in(mlp.bias), ddy(dy.values);
    Dev<double> gx(x.values.size()), gw(mlp.weight.values.size()), gb(mlp.bias.size());
    GinGrads r{FeatureMatrix(x.num_nodes, x.dim), FeatureMatrix(mlp.weight.num_nodes, mlp.weight.dim),
               std::vector<double>(mlp.bias.size()), 0.0};
    ok(gnna_gin_backward(ctx(), GNNA_F64, d.rp.get(), d.col.get(), t.rp.get(), t.col.get(), g.num_nodes, dx_in.get(),
                         x.dim, eps, dw_in.get(), mlp.weight.dim, db_in.get(), ddy.get(), gx.get(), gw.get(), gb.get(),
                         &r.deps));
    gx.to(r.dx.values.data(), r.dx.values.size());
    gw.to(r.dw.values.data(), r.dw.values.size());
    gb.to(r.db.data(), r.db.size());
    return r;
}

// ============================================================= decider
ModelInputs ModelInputs::from_graph(const CsrGraph& g, std::uint32_t dim) {
    if (dim == 0) throw DomainError("dim must be positive");
    const DegreeStats s = degree_stats(g);
    ModelInputs in;
    in.num_nodes = g.num_nodes;
    in.num_edges = g.num_edges();
    in.dim = dim;
    in.avg_degree = s.avg_degree;
    in.stddev_degree = s.stddev_degree;
    in.alpha = alpha_from_degrees(s.avg_degree, s.stddev_degree);
    return in;
}

double alpha_from_degrees(double avg, double sd) { return gnna_alpha_from_degrees(avg, sd); }

double wpt(const KernelParams& p) { return static_cast<double>(p.ngs) * p.dim / p.dw; }

std::uint64_t smem(const KernelParams& p) { return static_cast<std::uint64_t>(p.tpb / p.tpw) * p.dim * 4; }

std::uint32_t select_dw(std::uint32_t dim, std::uint32_t tpw) {
    std::uint32_t out = 0;
    decider_ok(gnna_select_dw(dim, tpw, &out), "select_dw");
    return out;
}

std::uint32_t select_ngs(std::uint32_t dw, std::uint32_t tpb, const ModelInputs& inputs) {
    const gnna_model_inputs c = to_c(inputs);
    std::uint32_t out = 0;
    decider_ok(gnna_select_ngs(dw, tpb, &c, &out), "select_ngs");
    return out;
}

double dp_size(std::uint64_t smem_bytes, double avg) {
    double out = 0.0;
    decider_ok(gnna_dp_size(smem_bytes, avg, &out), "dp_size");
    return out;
}

double estimate_latency(const KernelParams& p, const ModelInputs& inputs) {
    const gnna_params cp = to_c(p);
    const gnna_model_inputs ci = to_c(inputs);
    double out = 0.0;
    decider_ok(gnna_estimate_latency(&cp, &ci, &out), "estimate_latency");
    return out;
}

bool candidate_feasible(const KernelParams& p, const ModelInputs& inputs) {
    const gnna_params cp = to_c(p);
    const gnna_model_inputs ci = to_c(inputs);
    return gnna_candidate_feasible(&cp, &ci) != 0;
}

bool feasibility(const KernelParams& p, const ModelInputs& inputs) {
    const gnna_params cp = to_c(p);
    const gnna_model_inputs ci = to_c(inputs);
    return gnna_feasibility(&cp, &ci) != 0;
}

KernelParams auto_params(const ModelInputs& inputs) {
    const gnna_model_inputs c = to_c(inputs);
    gnna_params p{};
    decider_ok(gnna_auto_params(&c, &p), "auto_params");
    return from_c(p);
}

ParamCandidate search_params(const ModelInputs& inputs, std::uint32_t iterations, std::uint32_t population,
                             std::uint64_t seed, const SearchGrid& grid, SearchTrace* trace) {
    const gnna_model_inputs c = to_c(inputs);
    std::vector<double> tr(std::size_t(iterations) + 1);
    std::uint32_t tl = 0;
    gnna_params best{};
    double lat = 0.0;
    int feas = 0;
    decider_ok(gnna_search_params(&c, iterations, population, seed, grid.gs_values.data(),
                                  std::uint32_t(grid.gs_values.size()), grid.dw_values.data(),
                                  std::uint32_t(grid.dw_values.size()), grid.tpb_values.data(),
                                  std::uint32_t(grid.tpb_values.size()), &best, &lat, &feas, tr.data(), &tl),
               "search_params");
    if (trace) trace->best_per_iteration.assign(tr.begin(), tr.begin() + tl);
    ParamCandidate pc;
    pc.params = from_c(best);
    pc.estimated_latency = lat;
    pc.feasible = feas != 0;
    return pc;
}

// ============================================================ renumber
CommunityAssignment detect_communities(const CsrGraph& g) {
    const DevCsr d(g);
    Dev<std::uint32_t> com(g.num_nodes);
    CommunityAssignment ca;
    ok(gnna_detect_communities(ctx(), d.rp.get(), d.col.get(), g.num_nodes, com.get(), &ca.num_communities));
    ca.com_idx = com.host(g.num_nodes);
    return ca;
}

double modularity(const CsrGraph& g, const CommunityAssignment& ca) {
    if (ca.com_idx.size() != g.num_nodes) throw DomainError("modularity: assignment size mismatch");
    const DevCsr d(g);
    const Dev<std::uint32_t> com(ca.com_idx);
    double q = 0.0;
    ok(gnna_modularity(ctx(), d.rp.get(), d.col.get(), g.num_nodes, com.get(), ca.num_communities, &q));
    return q;
}

NodeMapping build_mapping(const CommunityAssignment& ca) {
    const std::size_t n = ca.com_idx.size();
    const Dev<std::uint32_t> com(ca.com_idx);
    Dev<std::uint32_t> o2n(n), n2o(n);
    ok(gnna_build_mapping(ctx(), com.get(), std::uint32_t(n), ca.num_communities, o2n.get(), n2o.get()));
    return NodeMapping{o2n.host(n), n2o.host(n)};
}

NodeMapping mapping_from_vector(std::vector<NodeId> old_to_new) {
    const std::size_t n = old_to_new.size();
    const Dev<std::uint32_t> v(old_to_new);
    Dev<std::uint32_t> o2n(n), n2o(n);
    ok(gnna_mapping_from_vector(ctx(), v.get(), std::uint32_t(n), o2n.get(), n2o.get()));
    return NodeMapping{std::move(old_to_new), n2o.host(n)};
}

CsrGraph apply_mapping(const CsrGraph& g, const NodeMapping& m) {
    if (m.old_to_new.size() != g.num_nodes || m.new_to_old.size() != g.num_nodes)
        throw DomainError("apply_mapping: mapping size does not match graph");
    const DevCsr d(g);
    const Dev<std::uint32_t> o2n(m.old_to_new), n2o(m.new_to_old);
    Dev<std::uint64_t> orp(std::size_t(g.num_nodes) + 1);
    Dev<std::uint32_t> ocol(g.num_edges());
    ok(gnna_apply_mapping_csr(ctx(), d.rp.get(), d.col.get(), g.num_nodes, o2n.get(), n2o.get(), orp.get(),
                              ocol.get()));
    CsrGraph out;
    out.num_nodes = g.num_nodes;
    out.row_ptr = orp.host(std::size_t(g.num_nodes) + 1);
    out.col_idx = ocol.host(g.num_edges());
    return out;
}

EdgeList apply_mapping(const EdgeList& el, const NodeMapping& m) {
    if (m.old_to_new.size() != el.num_nodes) throw DomainError("apply_mapping: mapping size does not match edge list");
    const Dev<std::uint32_t> e(flat_edges(el)), o2n(m.old_to_new);
    Dev<std::uint32_t> out(el.edges.size() * 2);
    ok(gnna_apply_mapping_edges(ctx(), e.get(), el.edges.size(), el.num_nodes, o2n.get(), out.get()));
    const auto h = out.host(el.edges.size() * 2);
    EdgeList r;
    r.num_nodes = el.num_nodes;
    r.edges.resize(el.edges.size());
    for (std::size_t i = 0; i < r.edges.size(); ++i) r.edges[i] = {h[2 * i], h[2 * i + 1]};
    return r;
}

bool should_reorder(const EdgeList& el) {
    const double threshold = std::floor(std::sqrt(static_cast<double>(el.num_nodes)) / 100.0);
    return std::sqrt(aes(el)) > threshold;
}

// ============================================================ pipeline
EdgeList planted_partition(std::uint32_t communities, std::uint32_t size, double p_in, double p_out, bool shuffle,
                           std::uint64_t seed) {
    if (communities == 0 || size == 0) throw DomainError("need at least one community of at least one node");
    if (!(p_in >= 0.0 && p_in <= 1.0) || !(p_out >= 0.0 && p_out <= 1.0))
        throw DomainError("edge probabilities must lie in [0, 1]");
    const std::uint64_t total = std::uint64_t(communities) * size;
    if (total > (1u << 16)) throw DomainError("generator samples all node pairs; limit is 65536 nodes");
    const NodeId n = static_cast<NodeId>(total);
    std::mt19937_64 rng(seed);
    EdgeList el;
    el.num_nodes = n;
    // every pair (i < j) in row-major order draws once
    for (NodeId i = 0; i < n; ++i)
        for (NodeId j = i + 1; j < n; ++j)
            if (draw_unit(rng) < ((i / size == j / size) ? p_in : p_out)) el.edges.emplace_back(i, j);
    if (shuffle) {
        std::vector<NodeId> perm(n);
        for (NodeId i = 0; i < n; ++i) perm[i] = i;
        for (NodeId i = n; i > 1; --i) std::swap(perm[i - 1], perm[draw_index(rng, i)]);
        for (auto& e : el.edges) e = {perm[e.first], perm[e.second]};
    }
    return el;
}

std::string edge_list_text(const EdgeList& el) {
    std::string s = "nodes " + std::to_string(el.num_nodes) + "\n";
    for (const auto& e : el.edges) s += std::to_string(e.first) + " " + std::to_string(e.second) + "\n";
    return s;
}

FeatureMatrix random_features(std::uint32_t num_nodes, std::uint32_t dim, std::uint64_t seed) {
    if (dim == 0) throw DomainError("dim must be positive");
    std::mt19937_64 rng(seed);
    FeatureMatrix x(num_nodes, dim);
    for (double& v : x.values) v = draw_unit(rng);
    return x;
}

StatsReport analyze(const EdgeList& el) {
    StatsReport r;
    r.num_nodes = el.num_nodes;
    r.num_edges = el.num_edges();
    r.aes = aes(el);
    r.sqrt_aes = std::sqrt(r.aes);
    r.threshold = std::floor(std::sqrt(static_cast<double>(el.num_nodes)) / 100.0);
    r.reorder = r.sqrt_aes > r.threshold;
    r.degrees = degree_stats(to_csr(el, true));
    return r;
}

ReorderResult reorder_edges(const EdgeList& el) {
    const CsrGraph g = to_csr(el, true);
    const CommunityAssignment ca = detect_communities(g);
    ReorderResult r;
    r.mapping = build_mapping(ca);
    r.num_communities = ca.num_communities;
    r.modularity = modularity(g, ca);
    r.aes_before = aes(el);
    r.aes_after = aes(apply_mapping(el, r.mapping));
    return r;
}

namespace {
// Device-resident CSR built from device edges (to_csr semantics).
struct DevGraph {
    uint32_t n = 0;
    uint64_t nnz = 0;
    Dev<std::uint64_t> rp;
    Dev<std::uint32_t> col;
    DevGraph(const std::uint32_t* d_edges, std::uint64_t e, std::uint32_t nodes, bool sym)
        : n(nodes), rp(std::size_t(nodes) + 1) {
        ok(gnna_to_csr(ctx(), n, d_edges, e, sym, rp.get(), nullptr, &nnz));
        col = Dev<std::uint32_t>(nnz);
        ok(gnna_to_csr(ctx(), n, d_edges, e, sym, rp.get(), col.get(), &nnz));
    }
};
}  // namespace

// pipeline.cpp:93-124 with every stage's data kept on the GPU (SURVEY
// §8(f)-3): the edge list is uploaded once, the symmetrised CSR, the
// community assignment, the mapping, the renumbered graph, the plan, the
// output and the verifying K4 oracle all stay in device memory; only the
// value-type results the API returns (stats, mapping, params, report,
// output) come back, plus the seeded features going up.
RunResult run_pipeline(const EdgeList& el, const RunConfig& config) {
    RunResult res;
    const std::uint64_t e = el.edges.size();
    if (e == 0) throw DomainError("no edges in the input");  // aes (analyze) on an empty list
    Dev<std::uint32_t> d_edges(flat_edges(el));
    // analyze (pipeline.cpp:69-79)
    res.stats.num_nodes = el.num_nodes;
    res.stats.num_edges = e;
    ok(gnna_aes(ctx(), d_edges.get(), e, &res.stats.aes));
    res.stats.sqrt_aes = std::sqrt(res.stats.aes);
    res.stats.threshold = std::floor(std::sqrt(static_cast<double>(el.num_nodes)) / 100.0);
    res.stats.reorder = res.stats.sqrt_aes > res.stats.threshold;
    std::unique_ptr<DevGraph> g = std::make_unique<DevGraph>(d_edges.get(), e, el.num_nodes, true);
    if (el.num_nodes == 0) throw DomainError("degree_stats: graph has no nodes");
    ok(gnna_degree_stats(ctx(), g->rp.get(), g->n, &res.stats.degrees.avg_degree, &res.stats.degrees.max_degree,
                         &res.stats.degrees.stddev_degree));
    res.reordered = config.force_reorder.value_or(res.stats.reorder);
    if (res.reordered) {  // reorder_edges (pipeline.cpp:81-91) + apply_mapping(el) (:101-102)
        const std::uint32_t n = el.num_nodes;
        Dev<std::uint32_t> com(n), o2n(n), n2o(n), moved(e * 2);
        ReorderResult r;
        ok(gnna_detect_communities(ctx(), g->rp.get(), g->col.get(), n, com.get(), &r.num_communities));
        ok(gnna_build_mapping(ctx(), com.get(), n, r.num_communities, o2n.get(), n2o.get()));
        ok(gnna_modularity(ctx(), g->rp.get(), g->col.get(), n, com.get(), r.num_communities, &r.modularity));
        r.aes_before = res.stats.aes;
        ok(gnna_apply_mapping_edges(ctx(), d_edges.get(), e, n, o2n.get(), moved.get()));
        ok(gnna_aes(ctx(), moved.get(), e, &r.aes_after));
        r.mapping.old_to_new = o2n.host(n);
        r.mapping.new_to_old = n2o.host(n);
        res.reorder = std::move(r);
        g = std::make_unique<DevGraph>(moved.get(), e, n, true);  // to_csr(work, true)
    }
    if (config.params) {
        res.params = *config.params;
        res.params.validate();
    } else {  // auto_params(ModelInputs::from_graph(g, dim)) on the device CSR
        if (config.dim == 0) throw DomainError("dim must be positive");
        gnna_model_inputs mi{};
        ok(gnna_model_inputs_from_graph(ctx(), g->rp.get(), g->n, config.dim, &mi));
        gnna_params p{};
        decider_ok(gnna_auto_params(&mi, &p), "auto_params");
        res.params = from_c(p);
    }
    const FeatureMatrix x = random_features(g->n, res.params.dim, config.seed);
    const Hubs hubs = make_hubs(g->rp.get(), g->col.get(), g->n, g->nnz, res.params.dim);
    const Dev<double> dx = upload_features(x, hubs);  // rows [0, n): x itself
    Dev<double> dy(x.values.size()), dref(x.values.size());
    EngineOptions opts;
    opts.workers = config.workers;
    opts.cache = config.cache;
    if (opts.cache) opts.cache->validate();
    const gnna_params c = to_c(res.params);
    const int strat = config.strategy == Strategy::NaiveAtomic ? GNNA_NAIVE_ATOMIC
                      : config.strategy == Strategy::UnitSync  ? GNNA_UNIT_SYNC
                                                               : GNNA_WARP_SHARED;
    const int mode = config.dim_mode == DimMode::Sequential ? GNNA_DIM_SEQUENTIAL : GNNA_DIM_CYCLIC;
    const PlanPtr plan = make_plan(g->rp.get(), g->col.get(), g->n, c, strat);
    if (hubs.k) {
        const PlanPtr hplan = make_plan(g->rp.get(), hubs.col2.get(), g->n, c, strat);
        aggregate_with_hubs(hplan.get(), hubs, g->n, res.params.dim, mode, dx.get(), dy.get());
    } else {
        aggregate_with_hubs(plan.get(), hubs, g->n, res.params.dim, mode, dx.get(), dy.get());
    }
    gnna_cost cost{};
    ok(gnna_cost_report(ctx(), plan.get(), mode, opts.transaction_line_bytes, opts.cache ? opts.cache->capacity : 0,
                        opts.cache ? opts.cache->line_size : 0, &cost));
    // pipeline.cpp:119-120: verify against the dense reference (K4 + features_close on the GPU)
    ok(gnna_aggregate_rows(ctx(), GNNA_F64, g->rp.get(), g->col.get(), g->n, res.params.dim, dx.get(), dref.get()));
    int close = 0;
    ok(gnna_features_close(ctx(), GNNA_F64, dy.get(), dref.get(), x.values.size(), 1e-12, &close));
    if (!close) throw InternalError("simulated aggregation deviates from the dense reference");
    res.report.atomic_ops = cost.atomic_ops;
    res.report.global_reads = cost.global_reads;
    res.report.global_writes = cost.global_writes;
    res.report.global_transactions = cost.global_transactions;
    res.report.shared_bytes_per_block = cost.shared_bytes_per_block;
    res.report.cache_hits = cost.cache_hits;
    res.report.cache_accesses = cost.cache_accesses;
    res.output = FeatureMatrix(g->n, res.params.dim);
    dy.to(res.output.values.data(), res.output.values.size());
    return res;
}

namespace b200 {
CallStats last_call_stats() { return t_stats; }
void clear_cache() { t_graphs.clear(); }
}  // namespace b200

}  // namespace gnnsim
