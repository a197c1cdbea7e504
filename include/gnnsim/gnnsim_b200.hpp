// gnnsim:: on B200 — the reference's C++ interface (proj/include/gnnsim/*.hpp
// of /root/reference), declared once here and implemented by
// libgnnsim_b200.so on top of the C-ABI in include/gnna.h.  Every compute
// entry point runs sm_100a kernels through libgnna.so; there is no CPU path.
//
// Source compatibility: the per-module headers next to this file
// (graph.hpp, schedule.hpp, memplan.hpp, engine.hpp, decider.hpp,
// renumber.hpp, pipeline.hpp, error.hpp, rand.hpp) include this one, so code
// written against the reference (its tests and acceptance gate) compiles
// unchanged.  Types keep the reference's field names, defaults and value
// semantics; functions keep names, argument meaning and exception types.
//
// Additions (no reference counterpart): gcn_layer_backward,
// gin_layer_backward, and set_device.
#pragma once

#include <algorithm>
#include <cstdint>
#include <iosfwd>
#include <map>
#include <optional>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace gnnsim {

// ===================================================== errors (error.hpp)
// Malformed input text; carries the 1-based line number when known.
class ParseError : public std::runtime_error {
public:
    ParseError(std::string msg, std::size_t line = 0)
        : std::runtime_error(line ? "line " + std::to_string(line) + ": " + msg : msg), line_(line) {}
    std::size_t line() const noexcept { return line_; }

private:
    std::size_t line_;
};

// Arguments outside an operation's domain.
class DomainError : public std::invalid_argument {
public:
    using std::invalid_argument::invalid_argument;
};

// File open / read / write failures.
class IoError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

// A checked invariant failed (e.g. verification against the dense oracle).
class InternalError : public std::logic_error {
public:
    using std::logic_error::logic_error;
};

// ============================================== deterministic draws (rand.hpp)
// Platform-independent draws over std::mt19937_64 (the distribution classes
// of <random> are implementation-defined).
inline std::size_t draw_index(std::mt19937_64& rng, std::size_t n) {
    const unsigned __int128 wide = static_cast<unsigned __int128>(rng()) * n;
    return static_cast<std::size_t>(wide >> 64);
}

inline double draw_unit(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

// ========================================================== graph (graph.hpp)
using NodeId = std::uint32_t;

struct EdgeList {
    NodeId num_nodes = 0;
    std::vector<std::pair<NodeId, NodeId>> edges;  // load order preserved
    std::size_t num_edges() const noexcept { return edges.size(); }
};

// Canonical CSR: each row ascending, no duplicate entries.
struct CsrGraph {
    NodeId num_nodes = 0;
    std::vector<std::uint64_t> row_ptr;  // num_nodes + 1 offsets
    std::vector<NodeId> col_idx;
    std::uint64_t num_edges() const noexcept { return col_idx.size(); }
    std::uint64_t degree(NodeId v) const { return row_ptr[v + 1] - row_ptr[v]; }
    std::span<const NodeId> neighbors(NodeId v) const {
        return {col_idx.data() + row_ptr[v], col_idx.data() + row_ptr[v + 1]};
    }
    bool operator==(const CsrGraph&) const = default;
};

// Dense row-major doubles: embeddings (num_nodes x dim) or weights (rows x cols).
struct FeatureMatrix {
    std::uint32_t num_nodes = 0;
    std::uint32_t dim = 0;
    std::vector<double> values;
    FeatureMatrix() = default;
    FeatureMatrix(std::uint32_t n, std::uint32_t d) : num_nodes(n), dim(d), values(std::size_t(n) * d, 0.0) {}
    double* row(std::uint32_t i) { return values.data() + std::size_t(i) * dim; }
    const double* row(std::uint32_t i) const { return values.data() + std::size_t(i) * dim; }
    double& at(std::uint32_t i, std::uint32_t j) { return row(i)[j]; }
    double at(std::uint32_t i, std::uint32_t j) const { return row(i)[j]; }
    bool operator==(const FeatureMatrix&) const = default;
};

struct DegreeStats {
    double avg_degree = 0.0;
    std::uint64_t max_degree = 0;
    double stddev_degree = 0.0;
};

EdgeList load_edge_list(std::istream& in);
EdgeList load_edge_list_file(const std::string& path);
CsrGraph to_csr(const EdgeList& el, bool symmetrize);  // GPU: gnna_to_csr
EdgeList to_edge_list(const CsrGraph& g);
DegreeStats degree_stats(const CsrGraph& g);           // GPU: gnna_degree_stats
double aes(const EdgeList& el);                        // GPU: gnna_aes
FeatureMatrix ones_features(std::uint32_t n, std::uint32_t dim);

// ==================================================== schedule (schedule.hpp)
struct KernelParams {
    std::uint32_t ngs = 16;
    std::uint32_t dw = 32;
    std::uint32_t tpb = 128;
    std::uint32_t tpw = 32;
    std::uint32_t dim = 16;
    std::uint32_t warps_per_block() const noexcept { return tpb / tpw; }
    void validate() const;  // DomainError on a violated invariant
    bool operator==(const KernelParams&) const = default;
};

// One workload unit: neighbours [begin, end) of node `target`.
struct NeighborGroup {
    std::uint32_t id = 0;
    NodeId target = 0;
    std::uint64_t begin = 0;
    std::uint64_t end = 0;
    std::uint64_t size() const noexcept { return end - begin; }
    bool operator==(const NeighborGroup&) const = default;
};

enum class DimMode { Sequential, Cyclic };

struct DimAssignment {
    DimMode mode = DimMode::Cyclic;
    std::vector<std::vector<std::uint32_t>> lanes;
};

struct WarpSchedule {
    std::vector<NeighborGroup> warps;
    std::uint32_t warp_per_block = 1;
    std::uint32_t num_warps() const noexcept { return static_cast<std::uint32_t>(warps.size()); }
    std::uint32_t num_blocks() const noexcept { return (num_warps() + warp_per_block - 1) / warp_per_block; }
    std::pair<std::uint32_t, std::uint32_t> block_range(std::uint32_t b) const noexcept {
        const std::uint32_t lo = b * warp_per_block;
        return {lo, std::min(lo + warp_per_block, num_warps())};
    }
};

std::vector<NeighborGroup> partition_neighbors(const CsrGraph& g, std::uint32_t ngs);  // GPU: K1
DimAssignment partition_dims(std::uint32_t dim, std::uint32_t dw, DimMode mode);
WarpSchedule map_warps(std::vector<NeighborGroup> groups, const KernelParams& params);

// ====================================================== memplan (memplan.hpp)
struct WarpPlanEntry {
    std::uint32_t slot = 0;
    NodeId node = 0;
    bool leader = false;
    bool operator==(const WarpPlanEntry&) const = default;
};

struct MemPlan {
    std::vector<WarpPlanEntry> entries;
    std::uint64_t shared_bytes_per_block = 0;
};

MemPlan build_mem_plan(const WarpSchedule& sched, const KernelParams& params);  // GPU: K2 (Algorithm 1)
std::map<NodeId, std::uint32_t> leaders_per_node(const MemPlan& plan, const WarpSchedule& sched);

// ======================================================== engine (engine.hpp)
enum class Strategy { NaiveAtomic, UnitSync, WarpShared };

struct CacheConfig {
    std::uint64_t capacity = 64 * 1024;
    std::uint64_t line_size = 128;
    void validate() const;
};

struct CostReport {
    std::uint64_t atomic_ops = 0;
    std::uint64_t global_reads = 0;
    std::uint64_t global_writes = 0;
    std::uint64_t global_transactions = 0;
    std::uint64_t shared_bytes_per_block = 0;
    std::uint64_t cache_hits = 0;
    std::uint64_t cache_accesses = 0;
    double cache_hit_rate() const noexcept {
        return cache_accesses ? static_cast<double>(cache_hits) / static_cast<double>(cache_accesses) : 0.0;
    }
};

struct EngineOptions {
    unsigned workers = 1;  // accepted for compatibility; the GPU result is worker-independent
    std::uint64_t transaction_line_bytes = 128;
    std::optional<CacheConfig> cache = CacheConfig{};
};

FeatureMatrix aggregate_oracle(const CsrGraph& g, const FeatureMatrix& x);  // GPU: K4
std::pair<FeatureMatrix, CostReport> aggregate_scheduled(const CsrGraph& g, const FeatureMatrix& x,
                                                         const KernelParams& params, Strategy strategy,
                                                         DimMode dim_mode, const EngineOptions& opts = {});  // GPU: K1+K2+K3+K8
bool features_close(const FeatureMatrix& a, const FeatureMatrix& b, double rel_tol);
std::uint64_t count_transactions(std::span<const std::uint64_t> addresses, std::uint64_t line = 128);
std::pair<std::uint64_t, std::uint64_t> simulate_cache(const CsrGraph& g, const WarpSchedule& sched,
                                                       const CacheConfig& cfg, std::uint32_t dim);  // GPU: K8 replay
FeatureMatrix gcn_layer(const CsrGraph& g, const FeatureMatrix& x, const FeatureMatrix& w,
                        bool add_self_loops = false);  // GPU: K5 + K6

struct AffineMap {
    FeatureMatrix weight;      // in_dim x out_dim
    std::vector<double> bias;  // out_dim
};

FeatureMatrix gin_layer(const CsrGraph& g, const FeatureMatrix& x, double eps, const AffineMap& mlp);  // GPU

// ---- additions: backward passes (no reference function)
struct GcnGrads {
    FeatureMatrix dx;  // n x in_dim
    FeatureMatrix dw;  // in_dim x out_dim
};
struct GinGrads {
    FeatureMatrix dx;
    FeatureMatrix dw;
    std::vector<double> db;
    double deps = 0.0;
};
// Gradients of L = <dy, layer(x)> w.r.t. the layer inputs.  The transposed
// adjacency is derived from g (g itself when g is symmetric).
GcnGrads gcn_layer_backward(const CsrGraph& g, const FeatureMatrix& x, const FeatureMatrix& w,
                            const FeatureMatrix& dy, bool add_self_loops = false);
GinGrads gin_layer_backward(const CsrGraph& g, const FeatureMatrix& x, double eps, const AffineMap& mlp,
                            const FeatureMatrix& dy);

// ====================================================== decider (decider.hpp)
struct ModelInputs {
    std::uint64_t num_nodes = 0;
    std::uint64_t num_edges = 0;
    std::uint32_t dim = 16;
    double avg_degree = 0.0;
    double stddev_degree = 0.0;
    std::uint32_t max_tpb = 1024;
    std::uint64_t smem_per_block = 96 * 1024;
    std::uint64_t capability = 4096;
    double alpha = 0.15;
    static ModelInputs from_graph(const CsrGraph& g, std::uint32_t dim);
};

double alpha_from_degrees(double avg_degree, double stddev_degree);

struct ParamCandidate {
    KernelParams params;
    double estimated_latency = 0.0;
    bool feasible = false;
};

double wpt(const KernelParams& p);
std::uint64_t smem(const KernelParams& p);
std::uint32_t select_dw(std::uint32_t dim, std::uint32_t tpw = 32);
std::uint32_t select_ngs(std::uint32_t dw, std::uint32_t tpb, const ModelInputs& inputs);
double dp_size(std::uint64_t smem_bytes, double avg_degree);
double estimate_latency(const KernelParams& p, const ModelInputs& inputs);
bool candidate_feasible(const KernelParams& p, const ModelInputs& inputs);
bool feasibility(const KernelParams& p, const ModelInputs& inputs);
KernelParams auto_params(const ModelInputs& inputs);

struct SearchGrid {
    std::vector<std::uint32_t> gs_values = {1, 2, 4, 8, 16, 32, 64};
    std::vector<std::uint32_t> dw_values = {8, 16, 32};
    std::vector<std::uint32_t> tpb_values = {32, 64, 128, 256};
};

struct SearchTrace {
    std::vector<double> best_per_iteration;
};

ParamCandidate search_params(const ModelInputs& inputs, std::uint32_t iterations = 15, std::uint32_t population = 32,
                             std::uint64_t seed = 1, const SearchGrid& grid = {}, SearchTrace* trace = nullptr);

// ==================================================== renumber (renumber.hpp)
struct CommunityAssignment {
    std::vector<std::uint32_t> com_idx;
    std::uint32_t num_communities = 0;
};

struct NodeMapping {
    std::vector<NodeId> old_to_new;
    std::vector<NodeId> new_to_old;
};

CommunityAssignment detect_communities(const CsrGraph& g);              // GPU: exact greedy merge
double modularity(const CsrGraph& g, const CommunityAssignment& ca);    // GPU
NodeMapping build_mapping(const CommunityAssignment& ca);               // GPU
NodeMapping mapping_from_vector(std::vector<NodeId> old_to_new);        // GPU
CsrGraph apply_mapping(const CsrGraph& g, const NodeMapping& m);        // GPU
EdgeList apply_mapping(const EdgeList& el, const NodeMapping& m);       // GPU
bool should_reorder(const EdgeList& el);

// ==================================================== pipeline (pipeline.hpp)
EdgeList planted_partition(std::uint32_t communities, std::uint32_t size, double p_in, double p_out, bool shuffle,
                           std::uint64_t seed);
std::string edge_list_text(const EdgeList& el);
FeatureMatrix random_features(std::uint32_t num_nodes, std::uint32_t dim, std::uint64_t seed);

struct StatsReport {
    std::uint64_t num_nodes = 0;
    std::uint64_t num_edges = 0;
    DegreeStats degrees;
    double aes = 0.0;
    double sqrt_aes = 0.0;
    double threshold = 0.0;
    bool reorder = false;
};

StatsReport analyze(const EdgeList& el);

struct ReorderResult {
    NodeMapping mapping;
    std::uint32_t num_communities = 0;
    double modularity = 0.0;
    double aes_before = 0.0;
    double aes_after = 0.0;
};

ReorderResult reorder_edges(const EdgeList& el);

struct RunConfig {
    std::string input;
    std::uint32_t dim = 16;
    std::optional<KernelParams> params;
    Strategy strategy = Strategy::WarpShared;
    DimMode dim_mode = DimMode::Cyclic;
    std::optional<CacheConfig> cache = CacheConfig{};
    std::optional<bool> force_reorder;
    std::uint64_t seed = 1;
    unsigned workers = 1;
};

struct RunResult {
    StatsReport stats;
    bool reordered = false;
    std::optional<ReorderResult> reorder;
    KernelParams params;
    CostReport report;
    FeatureMatrix output;
};

RunResult run_pipeline(const EdgeList& el, const RunConfig& config);

// ============================================================== device
// Selects the CUDA device for the calling thread's context (default: 0, or
// the GNNSIM_DEVICE environment variable).
void set_device(int device);

// ====================================================== B200 additions
// Not in the reference API: introspection of the drop-in's device cache and
// hub layout (see gnnsim_dropin.cpp).  GNNSIM_CACHE=0 / GNNSIM_HUB=0 turn
// them off.
namespace b200 {
struct CallStats {
    bool cache_hit = false;        // the graph's device CSR and plans were reused
    std::uint32_t hub_rows = 0;    // rows served from the L2-pinned hub block (0: layout off)
    std::uint64_t hub_edges = 0;   // CSR entries that gather a hub row
};
CallStats last_call_stats();       // of the calling thread's last aggregate_scheduled
void clear_cache();                // drops the calling thread's cached graphs
}  // namespace b200

}  // namespace gnnsim
