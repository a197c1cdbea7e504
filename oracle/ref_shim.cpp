// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (gnnsim, compiled from
// /root/reference/proj/src/*.cpp with -Dgnnsim=gnnsim_ref by oracle/Makefile).
// Exposes plain-pointer entry points so tests/ (ctypes) and bench.py's
// cpu_baseline / --impl reference arm can drive the reference's own code on the
// same inputs as the CUDA path.  Every function forwards to exactly one
// reference API call (cited), converting POD <-> std::vector value types.
//
// Status codes: 0 ok, 1 DomainError, 2 InternalError, 3 ParseError,
// 4 IoError, 5 other std::exception, 6 caller buffer too small.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "gnnsim/decider.hpp"
#include "gnnsim/engine.hpp"
#include "gnnsim/error.hpp"
#include "gnnsim/graph.hpp"
#include "gnnsim/memplan.hpp"
#include "gnnsim/pipeline.hpp"
#include "gnnsim/renumber.hpp"
#include "gnnsim/schedule.hpp"

using namespace gnnsim;  // renamed to gnnsim_ref by the Makefile's -D

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const DomainError& e) {
        g_err = e.what();
        return 1;
    } catch (const InternalError& e) {
        g_err = e.what();
        return 2;
    } catch (const ParseError& e) {
        g_err = e.what();
        return 3;
    } catch (const IoError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    } catch (...) {
        g_err = "caller buffer too small";
        return 6;
    }
}

struct TooSmall {};

CsrGraph view_csr(uint32_t n, const uint64_t* row_ptr, const uint32_t* col) {
    CsrGraph g;
    g.num_nodes = n;
    g.row_ptr.assign(row_ptr, row_ptr + n + 1);
    g.col_idx.assign(col, col + row_ptr[n]);
    return g;
}

EdgeList view_edges(uint32_t n, const uint32_t* edges, uint64_t e) {
    EdgeList el;
    el.num_nodes = n;
    el.edges.resize(e);
    for (uint64_t i = 0; i < e; ++i) el.edges[i] = {edges[2 * i], edges[2 * i + 1]};
    return el;
}

FeatureMatrix view_fm(uint32_t rows, uint32_t cols, const double* v) {
    FeatureMatrix m(rows, cols);
    std::memcpy(m.values.data(), v, sizeof(double) * rows * cols);
    return m;
}

KernelParams view_params(const uint32_t p[5]) {
    KernelParams k;
    k.ngs = p[0];
    k.dw = p[1];
    k.tpb = p[2];
    k.tpw = p[3];
    k.dim = p[4];
    return k;
}

void put_cost(const CostReport& c, uint64_t out[7]) {
    out[0] = c.atomic_ops;
    out[1] = c.global_reads;
    out[2] = c.global_writes;
    out[3] = c.global_transactions;
    out[4] = c.shared_bytes_per_block;
    out[5] = c.cache_hits;
    out[6] = c.cache_accesses;
}

// POD mirror of ModelInputs (decider.hpp:12-26); field order is the ABI.
struct PodInputs {
    uint64_t num_nodes, num_edges;
    uint32_t dim, max_tpb;
    double avg_degree, stddev_degree;
    uint64_t smem_per_block, capability;
    double alpha;
};

ModelInputs from_pod(const PodInputs* p) {
    ModelInputs in;
    in.num_nodes = p->num_nodes;
    in.num_edges = p->num_edges;
    in.dim = p->dim;
    in.max_tpb = p->max_tpb;
    in.avg_degree = p->avg_degree;
    in.stddev_degree = p->stddev_degree;
    in.smem_per_block = p->smem_per_block;
    in.capability = p->capability;
    in.alpha = p->alpha;
    return in;
}

void to_pod(const ModelInputs& in, PodInputs* p) {
    p->num_nodes = in.num_nodes;
    p->num_edges = in.num_edges;
    p->dim = in.dim;
    p->max_tpb = in.max_tpb;
    p->avg_degree = in.avg_degree;
    p->stddev_degree = in.stddev_degree;
    p->smem_per_block = in.smem_per_block;
    p->capability = in.capability;
    p->alpha = in.alpha;
}

void put_params(const KernelParams& k, uint32_t p[5]) {
    p[0] = k.ngs;
    p[1] = k.dw;
    p[2] = k.tpb;
    p[3] = k.tpw;
    p[4] = k.dim;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// graph.cpp:76 to_csr
int ref_to_csr(uint32_t n, const uint32_t* edges, uint64_t e, int symmetrize,
               uint64_t* row_ptr, uint32_t* col, uint64_t col_cap, uint64_t* nnz) {
    int rc = guard([&] {
        const CsrGraph g = to_csr(view_edges(n, edges, e), symmetrize != 0);
        *nnz = g.num_edges();
        if (g.num_edges() > col_cap) throw TooSmall{};
        std::memcpy(row_ptr, g.row_ptr.data(), sizeof(uint64_t) * (n + 1));
        std::memcpy(col, g.col_idx.data(), sizeof(uint32_t) * g.num_edges());
    });
    return rc;
}

// graph.cpp:122 aes
int ref_aes(uint32_t n, const uint32_t* edges, uint64_t e, double* out) {
    return guard([&] { *out = aes(view_edges(n, edges, e)); });
}

// renumber.cpp:198 should_reorder
int ref_should_reorder(uint32_t n, const uint32_t* edges, uint64_t e, int* out) {
    return guard([&] { *out = should_reorder(view_edges(n, edges, e)) ? 1 : 0; });
}

// graph.cpp:106 degree_stats
int ref_degree_stats(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                     double* avg, uint64_t* maxd, double* sd) {
    return guard([&] {
        const DegreeStats s = degree_stats(view_csr(n, row_ptr, col));
        *avg = s.avg_degree;
        *maxd = s.max_degree;
        *sd = s.stddev_degree;
    });
}

// schedule.cpp:7 KernelParams::validate
int ref_validate_params(const uint32_t p[5]) {
    return guard([&] { view_params(p).validate(); });
}

// schedule.cpp:16 partition_neighbors
int ref_partition_neighbors(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                            uint32_t ngs, uint64_t cap, uint64_t* num_groups,
                            uint32_t* ids, uint32_t* targets, uint64_t* begins,
                            uint64_t* ends) {
    return guard([&] {
        const auto groups = partition_neighbors(view_csr(n, row_ptr, col), ngs);
        *num_groups = groups.size();
        if (groups.size() > cap) throw TooSmall{};
        for (size_t i = 0; i < groups.size(); ++i) {
            ids[i] = groups[i].id;
            targets[i] = groups[i].target;
            begins[i] = groups[i].begin;
            ends[i] = groups[i].end;
        }
    });
}

// schedule.cpp:32 partition_dims -> flattened lanes: lane_ptr[dw+1], dims[]
int ref_partition_dims(uint32_t dim, uint32_t dw, int mode, uint32_t* lane_ptr,
                       uint32_t* dims) {
    return guard([&] {
        const DimAssignment da =
            partition_dims(dim, dw, mode == 0 ? DimMode::Sequential : DimMode::Cyclic);
        uint32_t k = 0;
        lane_ptr[0] = 0;
        for (size_t t = 0; t < da.lanes.size(); ++t) {
            for (uint32_t d : da.lanes[t]) dims[k++] = d;
            lane_ptr[t + 1] = k;
        }
    });
}

// memplan.cpp:9 build_mem_plan over groups {i, targets[i], i, i+1}
int ref_build_mem_plan(const uint32_t* targets, uint64_t num_groups, const uint32_t p[5],
                       uint32_t* slots, uint32_t* nodes, uint8_t* leaders,
                       uint64_t* smem_bytes) {
    return guard([&] {
        const KernelParams k = view_params(p);
        std::vector<NeighborGroup> groups(num_groups);
        for (uint64_t i = 0; i < num_groups; ++i)
            groups[i] = {static_cast<uint32_t>(i), targets[i], i, i + 1};
        const WarpSchedule s = map_warps(std::move(groups), k);
        const MemPlan plan = build_mem_plan(s, k);
        for (uint64_t i = 0; i < num_groups; ++i) {
            slots[i] = plan.entries[i].slot;
            nodes[i] = plan.entries[i].node;
            leaders[i] = plan.entries[i].leader ? 1 : 0;
        }
        *smem_bytes = plan.shared_bytes_per_block;
    });
}

// engine.cpp:200 aggregate_scheduled
int ref_aggregate_scheduled(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                            const double* x, const uint32_t p[5], int strategy,
                            int dim_mode, uint32_t workers, uint64_t line,
                            int cache_on, uint64_t cache_cap, uint64_t cache_line,
                            double* y, uint64_t cost[7]) {
    return guard([&] {
        const KernelParams k = view_params(p);
        EngineOptions opts;
        opts.workers = workers;
        opts.transaction_line_bytes = line;
        if (cache_on)
            opts.cache = CacheConfig{cache_cap, cache_line};
        else
            opts.cache.reset();
        const Strategy s = strategy == 0   ? Strategy::NaiveAtomic
                           : strategy == 1 ? Strategy::UnitSync
                                           : Strategy::WarpShared;
        const auto [out, rep] =
            aggregate_scheduled(view_csr(n, row_ptr, col), view_fm(n, k.dim, x), k, s,
                                dim_mode == 0 ? DimMode::Sequential : DimMode::Cyclic, opts);
        std::memcpy(y, out.values.data(), sizeof(double) * out.values.size());
        put_cost(rep, cost);
    });
}

// engine.cpp:149 aggregate_oracle
int ref_aggregate_oracle(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                         const double* x, uint32_t dim, double* y) {
    return guard([&] {
        const FeatureMatrix out =
            aggregate_oracle(view_csr(n, row_ptr, col), view_fm(n, dim, x));
        std::memcpy(y, out.values.data(), sizeof(double) * out.values.size());
    });
}

// engine.cpp:174 count_transactions
int ref_count_transactions(const uint64_t* addr, uint64_t k, uint64_t line,
                           uint64_t* out) {
    return guard([&] {
        *out = count_transactions(std::span<const uint64_t>(addr, k), line);
    });
}

// engine.cpp:185 simulate_cache over map_warps(partition_neighbors(g, ngs), p)
int ref_simulate_cache(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                       const uint32_t p[5], uint64_t cache_cap, uint64_t cache_line,
                       uint32_t dim, uint64_t* hits, uint64_t* accesses) {
    return guard([&] {
        const CsrGraph g = view_csr(n, row_ptr, col);
        const KernelParams k = view_params(p);
        const WarpSchedule s = map_warps(partition_neighbors(g, k.ngs), k);
        const auto [h, a] = simulate_cache(g, s, CacheConfig{cache_cap, cache_line}, dim);
        *hits = h;
        *accesses = a;
    });
}

// engine.cpp:373 gcn_layer
int ref_gcn_layer(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                  const double* x, uint32_t in_dim, const double* w, uint32_t out_dim,
                  int self_loops, double* y) {
    return guard([&] {
        const FeatureMatrix out =
            gcn_layer(view_csr(n, row_ptr, col), view_fm(n, in_dim, x),
                      view_fm(in_dim, out_dim, w), self_loops != 0);
        std::memcpy(y, out.values.data(), sizeof(double) * out.values.size());
    });
}

// engine.cpp:384 gin_layer
int ref_gin_layer(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                  const double* x, uint32_t in_dim, double eps, const double* w,
                  uint32_t out_dim, const double* b, double* y) {
    return guard([&] {
        AffineMap mlp;
        mlp.weight = view_fm(in_dim, out_dim, w);
        mlp.bias.assign(b, b + out_dim);
        const FeatureMatrix out =
            gin_layer(view_csr(n, row_ptr, col), view_fm(n, in_dim, x), eps, mlp);
        std::memcpy(y, out.values.data(), sizeof(double) * out.values.size());
    });
}

// renumber.cpp:31 detect_communities
int ref_detect_communities(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                           uint32_t* com, uint32_t* ncom) {
    return guard([&] {
        const CommunityAssignment ca = detect_communities(view_csr(n, row_ptr, col));
        std::memcpy(com, ca.com_idx.data(), sizeof(uint32_t) * n);
        *ncom = ca.num_communities;
    });
}

// renumber.cpp:106 modularity
int ref_modularity(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                   const uint32_t* com, uint32_t ncom, double* q) {
    return guard([&] {
        CommunityAssignment ca;
        ca.com_idx.assign(com, com + n);
        ca.num_communities = ncom;
        *q = modularity(view_csr(n, row_ptr, col), ca);
    });
}

// renumber.cpp:128 build_mapping
int ref_build_mapping(uint32_t n, const uint32_t* com, uint32_t ncom, uint32_t* o2n,
                      uint32_t* n2o) {
    return guard([&] {
        CommunityAssignment ca;
        ca.com_idx.assign(com, com + n);
        ca.num_communities = ncom;
        const NodeMapping m = build_mapping(ca);
        std::memcpy(o2n, m.old_to_new.data(), sizeof(uint32_t) * n);
        std::memcpy(n2o, m.new_to_old.data(), sizeof(uint32_t) * n);
    });
}

// renumber.cpp:148 mapping_from_vector
int ref_mapping_from_vector(uint32_t n, const uint32_t* v, uint32_t* o2n, uint32_t* n2o) {
    return guard([&] {
        const NodeMapping m = mapping_from_vector(std::vector<NodeId>(v, v + n));
        std::memcpy(o2n, m.old_to_new.data(), sizeof(uint32_t) * n);
        std::memcpy(n2o, m.new_to_old.data(), sizeof(uint32_t) * n);
    });
}

// renumber.cpp:162 apply_mapping (CSR)
int ref_apply_mapping_csr(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                          const uint32_t* o2n, const uint32_t* n2o, uint64_t* out_row_ptr,
                          uint32_t* out_col) {
    return guard([&] {
        NodeMapping m;
        m.old_to_new.assign(o2n, o2n + n);
        m.new_to_old.assign(n2o, n2o + n);
        const CsrGraph g = apply_mapping(view_csr(n, row_ptr, col), m);
        std::memcpy(out_row_ptr, g.row_ptr.data(), sizeof(uint64_t) * (n + 1));
        std::memcpy(out_col, g.col_idx.data(), sizeof(uint32_t) * g.num_edges());
    });
}

// renumber.cpp:187 apply_mapping (EdgeList)
int ref_apply_mapping_edges(uint32_t n, const uint32_t* edges, uint64_t e,
                            const uint32_t* o2n, const uint32_t* n2o, uint32_t* out) {
    return guard([&] {
        NodeMapping m;
        m.old_to_new.assign(o2n, o2n + n);
        m.new_to_old.assign(n2o, n2o + n);
        const EdgeList el = apply_mapping(view_edges(n, edges, e), m);
        for (uint64_t i = 0; i < e; ++i) {
            out[2 * i] = el.edges[i].first;
            out[2 * i + 1] = el.edges[i].second;
        }
    });
}

// pipeline.cpp:57 random_features
int ref_random_features(uint32_t n, uint32_t dim, uint64_t seed, double* out) {
    return guard([&] {
        const FeatureMatrix x = random_features(n, dim, seed);
        std::memcpy(out, x.values.data(), sizeof(double) * x.values.size());
    });
}

// pipeline.cpp:14 planted_partition
int ref_planted_partition(uint32_t communities, uint32_t size, double p_in, double p_out,
                          int shuffle, uint64_t seed, uint64_t cap, uint32_t* edges,
                          uint64_t* num_edges, uint32_t* num_nodes) {
    return guard([&] {
        const EdgeList el =
            planted_partition(communities, size, p_in, p_out, shuffle != 0, seed);
        *num_edges = el.edges.size();
        *num_nodes = el.num_nodes;
        if (el.edges.size() > cap) throw TooSmall{};
        for (size_t i = 0; i < el.edges.size(); ++i) {
            edges[2 * i] = el.edges[i].first;
            edges[2 * i + 1] = el.edges[i].second;
        }
    });
}

// pipeline.cpp:81 reorder_edges
int ref_reorder_edges(uint32_t n, const uint32_t* edges, uint64_t e, uint32_t* o2n,
                      uint32_t* n2o, uint32_t* ncom, double* q, double* aes_before,
                      double* aes_after) {
    return guard([&] {
        const ReorderResult r = reorder_edges(view_edges(n, edges, e));
        std::memcpy(o2n, r.mapping.old_to_new.data(), sizeof(uint32_t) * n);
        std::memcpy(n2o, r.mapping.new_to_old.data(), sizeof(uint32_t) * n);
        *ncom = r.num_communities;
        *q = r.modularity;
        *aes_before = r.aes_before;
        *aes_after = r.aes_after;
    });
}

// pipeline.cpp:93-124 run_pipeline.  force_reorder: -1 absent (the AES rule
// decides), 0 / 1 forced; params_in[0] == 0: auto_params; cache_capacity 0:
// no cache replay, else CacheConfig{capacity, line}.  Outputs: the stats,
// the reorder result (o2n, ncom, Q, AES before/after), the params used, the
// CostReport (7 counters, engine.hpp order) and the n x dim output.
int ref_run_pipeline(uint32_t n, const uint32_t* edges, uint64_t e, uint32_t dim, const uint32_t params_in[5],
                     int strategy, int dim_mode, int force_reorder, uint64_t seed, uint64_t cache_capacity,
                     uint64_t cache_line, unsigned workers, int* reordered, uint32_t* o2n, uint32_t* ncom,
                     double* q, double* aes, uint32_t params_out[5], uint64_t report[7], double* out) {
    return guard([&] {
        RunConfig cfg;
        cfg.dim = dim;
        if (params_in[0]) {
            KernelParams k;
            k.ngs = params_in[0];
            k.dw = params_in[1];
            k.tpb = params_in[2];
            k.tpw = params_in[3];
            k.dim = params_in[4];
            cfg.params = k;
        }
        cfg.strategy = static_cast<Strategy>(strategy);
        cfg.dim_mode = static_cast<DimMode>(dim_mode);
        if (cache_capacity) cfg.cache = CacheConfig{cache_capacity, cache_line};
        else cfg.cache = std::nullopt;
        if (force_reorder >= 0) cfg.force_reorder = force_reorder != 0;
        cfg.seed = seed;
        cfg.workers = workers;
        const RunResult r = run_pipeline(view_edges(n, edges, e), cfg);
        *reordered = r.reordered ? 1 : 0;
        aes[0] = r.stats.aes;
        if (r.reorder) {
            std::memcpy(o2n, r.reorder->mapping.old_to_new.data(), sizeof(uint32_t) * n);
            *ncom = r.reorder->num_communities;
            *q = r.reorder->modularity;
            aes[1] = r.reorder->aes_before;
            aes[2] = r.reorder->aes_after;
        }
        put_params(r.params, params_out);
        report[0] = r.report.atomic_ops;
        report[1] = r.report.global_reads;
        report[2] = r.report.global_writes;
        report[3] = r.report.global_transactions;
        report[4] = r.report.shared_bytes_per_block;
        report[5] = r.report.cache_hits;
        report[6] = r.report.cache_accesses;
        std::memcpy(out, r.output.values.data(), sizeof(double) * r.output.values.size());
    });
}

// decider.cpp:26 ModelInputs::from_graph
int ref_model_inputs(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                     uint32_t dim, PodInputs* out) {
    return guard([&] { to_pod(ModelInputs::from_graph(view_csr(n, row_ptr, col), dim), out); });
}

// decider.cpp:20 alpha_from_degrees
double ref_alpha_from_degrees(double avg, double sd) { return alpha_from_degrees(avg, sd); }

// decider.cpp:47 select_dw
int ref_select_dw(uint32_t dim, uint32_t tpw, uint32_t* out) {
    return guard([&] { *out = select_dw(dim, tpw); });
}

// decider.cpp:53 select_ngs
int ref_select_ngs(uint32_t dw, uint32_t tpb, const PodInputs* in, uint32_t* out) {
    return guard([&] { *out = select_ngs(dw, tpb, from_pod(in)); });
}

// decider.cpp:64 dp_size
int ref_dp_size(uint64_t smem_bytes, double avg, double* out) {
    return guard([&] { *out = dp_size(smem_bytes, avg); });
}

// decider.cpp:70 estimate_latency
int ref_estimate_latency(const uint32_t p[5], const PodInputs* in, double* out) {
    return guard([&] { *out = estimate_latency(view_params(p), from_pod(in)); });
}

// decider.cpp:83/88 candidate_feasible, feasibility
int ref_feasible(const uint32_t p[5], const PodInputs* in, int* cand, int* feas) {
    return guard([&] {
        *cand = candidate_feasible(view_params(p), from_pod(in)) ? 1 : 0;
        *feas = feasibility(view_params(p), from_pod(in)) ? 1 : 0;
    });
}

// decider.cpp:99 auto_params
int ref_auto_params(const PodInputs* in, uint32_t p[5]) {
    return guard([&] { put_params(auto_params(from_pod(in)), p); });
}

// decider.cpp:138 search_params
int ref_search_params(const PodInputs* in, uint32_t iterations, uint32_t population,
                      uint64_t seed, const uint32_t* gs, uint32_t ngs_n, const uint32_t* dw,
                      uint32_t ndw, const uint32_t* tpb, uint32_t ntpb, uint32_t p[5],
                      double* latency, int* feasible, double* trace, uint32_t* trace_len) {
    return guard([&] {
        SearchGrid grid;
        grid.gs_values.assign(gs, gs + ngs_n);
        grid.dw_values.assign(dw, dw + ndw);
        grid.tpb_values.assign(tpb, tpb + ntpb);
        SearchTrace tr;
        const ParamCandidate c =
            search_params(from_pod(in), iterations, population, seed, grid, &tr);
        put_params(c.params, p);
        *latency = c.estimated_latency;
        *feasible = c.feasible ? 1 : 0;
        *trace_len = static_cast<uint32_t>(tr.best_per_iteration.size());
        for (size_t i = 0; i < tr.best_per_iteration.size(); ++i)
            trace[i] = tr.best_per_iteration[i];
    });
}

}  // extern "C"

extern "C" {
// CPU baseline for bench.py: builds the reference value types once, then times
// `reps` calls of the reference's own aggregate_scheduled (engine.cpp:200)
// with std::chrono::steady_clock; only the reference call is inside the clock.
int ref_time_aggregate_scheduled(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                                 const double* x, const uint32_t p[5], int strategy,
                                 int dim_mode, uint32_t workers, uint32_t reps,
                                 double* y, double* seconds) {
    return guard([&] {
        const KernelParams k = view_params(p);
        EngineOptions opts;
        opts.workers = workers;
        opts.cache.reset();
        const Strategy s = strategy == 0   ? Strategy::NaiveAtomic
                           : strategy == 1 ? Strategy::UnitSync
                                           : Strategy::WarpShared;
        const CsrGraph g = view_csr(n, row_ptr, col);
        const FeatureMatrix fx = view_fm(n, k.dim, x);
        const auto mode = dim_mode == 0 ? DimMode::Sequential : DimMode::Cyclic;
        double total = 0.0;
        for (uint32_t r = 0; r < reps; ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            const auto [out, rep] = aggregate_scheduled(g, fx, k, s, mode, opts);
            const auto t1 = std::chrono::steady_clock::now();
            total += std::chrono::duration<double>(t1 - t0).count();
            if (r + 1 == reps && y)
                std::memcpy(y, out.values.data(), sizeof(double) * out.values.size());
        }
        *seconds = total;
    });
}

// Same for aggregate_oracle (engine.cpp:149), single-threaded by design.
int ref_time_aggregate_oracle(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                              const double* x, uint32_t dim, uint32_t reps, double* seconds) {
    return guard([&] {
        const CsrGraph g = view_csr(n, row_ptr, col);
        const FeatureMatrix fx = view_fm(n, dim, x);
        double total = 0.0;
        for (uint32_t r = 0; r < reps; ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            const FeatureMatrix out = aggregate_oracle(g, fx);
            const auto t1 = std::chrono::steady_clock::now();
            total += std::chrono::duration<double>(t1 - t0).count();
        }
        *seconds = total;
    });
}

}  // extern "C"
