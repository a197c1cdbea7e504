/* gnna.h — the C-ABI boundary of the B200 GNNAdvisor aggregation runtime.
 *
 * Plain pointers and sizes only: no C++ or torch types cross this line.  Every
 * device-pointer entry point is stream-ordered on the context's stream
 * (gnna_set_stream; default: the legacy default stream) and returns without
 * synchronising unless it returns a host scalar.  Each entry names the
 * reference interface (/root/reference/proj, namespace gnnsim) it replaces;
 * the C++ drop-in (the include/gnnsim/ headers, libgnnsim_b200.so) is implemented on
 * top of exactly these calls.
 *
 * Errors mirror the reference's exception taxonomy (error.hpp:9-38):
 * GNNA_ERR_DOMAIN <-> DomainError (with the reference's message text),
 * GNNA_ERR_INTERNAL <-> InternalError.  CUDA/OOM failures have their own
 * codes.  gnna_last_error(ctx) returns the message of the last failure on ctx.
 *
 * There is no CPU fallback: every compute entry point runs CUDA kernels built
 * for sm_100a; without a usable device gnna_create fails with GNNA_ERR_CUDA.
 */
#ifndef GNNA_H
#define GNNA_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define GNNA_API __attribute__((visibility("default")))
#else
#define GNNA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef int gnna_status;
#define GNNA_OK 0
#define GNNA_ERR_DOMAIN 1
#define GNNA_ERR_INTERNAL 2
#define GNNA_ERR_CUDA 3
#define GNNA_ERR_OOM 4

/* engine.hpp:21 Strategy */
#define GNNA_NAIVE_ATOMIC 0
#define GNNA_UNIT_SYNC 1
#define GNNA_WARP_SHARED 2
/* schedule.hpp:42 DimMode */
#define GNNA_DIM_SEQUENTIAL 0
#define GNNA_DIM_CYCLIC 1
/* element type of feature matrices */
#define GNNA_F32 0
#define GNNA_F64 1

/* schedule.hpp:14-27 KernelParams (same field meaning; tpw fixed at 32). */
typedef struct {
    uint32_t ngs, dw, tpb, tpw, dim;
} gnna_params;

/* engine.hpp:30-53 CostReport */
typedef struct {
    uint64_t atomic_ops, global_reads, global_writes, global_transactions;
    uint64_t shared_bytes_per_block, cache_hits, cache_accesses;
} gnna_cost;

/* decider.hpp:12-26 ModelInputs (field order is the ABI). */
typedef struct {
    uint64_t num_nodes, num_edges;
    uint32_t dim, max_tpb;
    double avg_degree, stddev_degree;
    uint64_t smem_per_block, capability;
    double alpha;
} gnna_model_inputs;

typedef struct gnna_ctx gnna_ctx;
typedef struct gnna_plan gnna_plan;

/* ------------------------------------------------------------ context --- */
GNNA_API gnna_status gnna_create(int device, gnna_ctx** out);
GNNA_API void gnna_destroy(gnna_ctx* ctx);
GNNA_API gnna_status gnna_set_stream(gnna_ctx* ctx, void* cuda_stream);
GNNA_API void* gnna_get_stream(const gnna_ctx* ctx);
GNNA_API gnna_status gnna_synchronize(gnna_ctx* ctx);
GNNA_API const char* gnna_last_error(const gnna_ctx* ctx);
/* L2 residency for the gather's hot rows (B200: 126 MB L2).  Marks
 * [base, base + bytes) as an access-policy window on the context's stream:
 * hits persist in a set-aside L2 region (sized to the window, capped at the
 * device's persisting maximum), misses stream.  With rows numbered by
 * descending degree (the power-law hubs first), the window holds the rows
 * the aggregation re-reads most.  bytes == 0 clears the window and resets the
 * persisting lines.  *applied (may be NULL) receives the window size used. */
GNNA_API gnna_status gnna_set_l2_window(gnna_ctx* ctx, const void* base, uint64_t bytes, double hit_ratio,
                                        uint64_t* applied);
GNNA_API const char* gnna_version(void);
/* Number of kernels this library has launched on ctx (for bench.py). */
GNNA_API uint64_t gnna_launch_count(const gnna_ctx* ctx);

/* Device memory for hosts that do not link the CUDA runtime themselves (the
 * gnnsim:: C++ drop-in).  Allocation is stream-ordered on ctx's stream;
 * gnna_copy_to_host synchronises the stream before returning.  Host buffers
 * may be pageable: copies of 4 MiB and more from / to pageable memory go
 * through the context's pinned bounce buffers (8 MiB chunks, host threads
 * copying one chunk while the DMA engine moves the previous one); the host
 * source of gnna_copy_to_device is free again when it returns. */
GNNA_API gnna_status gnna_device_alloc(gnna_ctx* ctx, size_t bytes, void** out);
GNNA_API gnna_status gnna_device_free(gnna_ctx* ctx, void* p);
GNNA_API gnna_status gnna_copy_to_device(gnna_ctx* ctx, void* d_dst, const void* h_src, size_t bytes);
GNNA_API gnna_status gnna_copy_to_host(gnna_ctx* ctx, void* h_dst, const void* d_src, size_t bytes);

/* -------------------------------------------------- parameter domain --- */
/* schedule.cpp:7-14 KernelParams::validate — same order, same messages. */
GNNA_API gnna_status gnna_validate_params(gnna_ctx* ctx, const gnna_params* p);

/* ------------------------------------------------ preprocessing (K1/K2) */
/* Number of workload units: sum_v ceil(deg(v)/ngs) (schedule.cpp:16-30). */
GNNA_API gnna_status gnna_count_groups(gnna_ctx* ctx, const uint64_t* d_row_ptr, uint32_t n,
                              uint32_t ngs, uint64_t* num_groups);
/* schedule.hpp:76 partition_neighbors: unit u covers CSR range
 * [d_part_ptr[u], d_part_ptr[u+1]) of node d_part2node[u] (NeighborGroup
 * {id=u, target, begin, end}; begin_{u+1} == end_u, so G+1 offsets suffice). */
GNNA_API gnna_status gnna_partition_neighbors(gnna_ctx* ctx, const uint64_t* d_row_ptr, uint32_t n,
                                     uint32_t ngs, uint64_t* d_part_ptr,
                                     uint32_t* d_part2node);
/* memplan.hpp:43 build_mem_plan (Algorithm 1) for warps targeting
 * d_part2node[0..G): slot (node_shared_addr, slot index) and leader
 * (unit_leader) per unit.  GNNA_ERR_DOMAIN when a node's units are not
 * consecutive (memplan.cpp:15-29).  *shared_bytes = wpb*dim*4. */
GNNA_API gnna_status gnna_build_mem_plan(gnna_ctx* ctx, const uint32_t* d_part2node,
                                uint64_t num_groups, const gnna_params* p, uint8_t* d_slot,
                                uint8_t* d_leader, uint64_t* shared_bytes);

/* ------------------------------------------------------------- plans --- */
/* Device-resident schedule for rows [row_begin, row_end) of a CSR graph:
 * K1 units, K2 Algorithm-1 slots/leaders, run/carry layout.  The reference
 * rebuilds this inside every aggregate_scheduled call (engine.cpp:213-221);
 * here it is built once and reused.  The plan keeps pointers to d_row_ptr and
 * d_col, which must outlive it.  Strategy NaiveAtomic/UnitSync flush every
 * unit on its own, WarpShared per Algorithm-1 run.
 * Streams: the plan's arrays are allocated (stream-ordered) on the context's
 * stream at creation and freed on that stream by gnna_plan_destroy, so that
 * stream must outlive the plan.  A plan holds mutable carry scratch: do not
 * run aggregations of ONE plan on two streams concurrently (one plan per
 * stream; plans over the same CSR are cheap). */
GNNA_API gnna_status gnna_plan_create(gnna_ctx* ctx, const uint64_t* d_row_ptr, const uint32_t* d_col,
                             uint32_t n, uint32_t row_begin, uint32_t row_end,
                             const gnna_params* p, int strategy, gnna_plan** out);
GNNA_API void gnna_plan_destroy(gnna_plan* plan);
GNNA_API gnna_status gnna_plan_info(const gnna_plan* plan, uint64_t* num_groups, uint64_t* num_runs,
                           uint64_t* num_split_nodes, uint64_t* num_carries);
/* Device arrays of the plan (valid while the plan lives). */
GNNA_API gnna_status gnna_plan_arrays(const gnna_plan* plan, const uint64_t** d_part_ptr,
                             const uint32_t** d_part2node, const uint8_t** d_slot,
                             const uint8_t** d_leader);

/* ------------------------------------------------- aggregation (K3) --- */
/* engine.hpp:71 aggregate_scheduled, values only: y[v] = sum_{u in N(v)} x[u]
 * for the plan's rows, evaluated in the reference's summation tree (unit
 * partials in CSR order -> Algorithm-1 run sums in unit order -> ordered
 * cross-block combine).  GNNA_F64 is bitwise equal to the reference;
 * GNNA_F32 follows the same tree in fp32.  x, y: n x dim row-major. */
GNNA_API gnna_status gnna_aggregate(gnna_ctx* ctx, const gnna_plan* plan, int dtype, int dim_mode,
                           const void* d_x, void* d_y);
/* Options of gnna_aggregate_ex: the fused forms the layer entry points need
 * (engine.cpp:338-408).  For each output row v of the plan:
 *   y[v] = relu?( row_scale[v] * ( sum_{u in N(v)} node_weight[u] * x[u]
 *                                  + self_weight[v] * x[v] ) )  (masked)
 * node_weight is per source node (F32 only; NULL = all ones; GCN: norm);
 * self_weight NULL uses the constant alpha (0 = no self term); row_scale NULL
 * = 1; mask (same shape/dtype as y) zeroes y where mask <= 0 (ReLU backward).
 * dim 0 = the plan's params.dim; any other width reuses the plan's schedule.
 * With node weights and >= 4 edges per row, x is first scaled row by row into
 * a stream-ordered scratch copy (n x dim floats) that the gather reads; the
 * self term still reads x, and an L2 access-policy window on ctx's stream that
 * covers rows of x is moved to the same rows of the copy for the launch.  Each
 * term is then rn(node_weight[u] * x[u]) added in CSR order (the GCN layer's
 * rounding), instead of one fmaf per edge (GNNA_PRESCALE=0). */
typedef struct {
    uint32_t dim;
    const float* node_weight;
    const float* self_weight;
    double alpha;
    const float* row_scale;
    int relu;
    const void* mask;
} gnna_agg_opts;
GNNA_API gnna_status gnna_aggregate_ex(gnna_ctx* ctx, const gnna_plan* plan, int dtype, int dim_mode,
                              const void* d_x, void* d_y, const gnna_agg_opts* opts);

/* Multi-GPU row sharding with the all-gather fused into the aggregation
 * (SURVEY §8(e) "fused target"; replaces aggregate + the per-layer
 * ncclBroadcast-per-owner all-gather of the reference's sharded use).  Same
 * as gnna_aggregate_ex on this rank's row-slice plan, and every final row
 * value is ALSO written at the same row offset into
 *   - each peer_y[i] (i < n_peer <= GNNA_MAX_PEERS): device pointers of the
 *     other ranks' replicas of y, P2P-mapped into this context (NVLink stores
 *     overlapped with the gather), or
 *   - mc_y, when non-NULL: the NVLS multicast address bound to every rank's
 *     replica of y (multimem.st; the switch writes all copies, this rank's
 *     included, and d_y is not written separately).
 * The caller orders the peers' reads after every rank's kernel (a stream-
 * ordered cross-rank barrier), and this rank's stores after the peers'
 * reads of the previous contents.  Rows outside the plan are never written.
 * Node weights (opts->node_weight: GCN's gathered norm[u]) take the pre-scaled
 * gather of gnna_aggregate_ex (any width; the replicas get the same bits); with
 * GNNA_PRESCALE=0 or < 4 edges per row, only fp32 rows of at most one 16-byte
 * chunk per lane (GNNA_ERR_DOMAIN otherwise). */
#define GNNA_MAX_PEERS 7
GNNA_API gnna_status gnna_aggregate_fanout(gnna_ctx* ctx, const gnna_plan* plan, int dtype, int dim_mode,
                                           const void* d_x, void* d_y, const gnna_agg_opts* opts,
                                           void* const* peer_y, uint32_t n_peer, void* mc_y);

/* engine.hpp:30-53 + engine.cpp:242-289: the integer CostReport of
 * aggregate_scheduled for this plan (K8).  cache_line == 0 disables the LRU
 * replay (EngineOptions::cache = nullopt). */
GNNA_API gnna_status gnna_cost_report(gnna_ctx* ctx, const gnna_plan* plan, int dim_mode,
                             uint64_t line_bytes, uint64_t cache_capacity, uint64_t cache_line,
                             gnna_cost* out);
/* engine.hpp:77 simulate_cache over the plan's schedule. */
GNNA_API gnna_status gnna_simulate_cache(gnna_ctx* ctx, const gnna_plan* plan, uint64_t cache_capacity,
                                uint64_t cache_line, uint32_t dim, uint64_t* hits,
                                uint64_t* accesses);

/* engine.hpp:77 simulate_cache over an explicit warp schedule (WarpSchedule:
 * warp w covers col[d_begin[w] .. d_end[w]), blocks of warps_per_block
 * consecutive warps).  Same replay as gnna_simulate_cache; used by the C++
 * drop-in, whose callers may hand in any schedule. */
GNNA_API gnna_status gnna_simulate_cache_ranges(gnna_ctx* ctx, const uint32_t* d_col,
                                       const uint64_t* d_begin, const uint64_t* d_end,
                                       uint64_t num_warps, uint32_t warps_per_block,
                                       uint64_t cache_capacity, uint64_t cache_line,
                                       uint32_t dim, uint64_t* hits, uint64_t* accesses);

/* engine.hpp:78 features_close on device data (same element count, same
 * dtype): *close = 1 iff no element has |a-b| > rel_tol * max(|a|,|b|). */
GNNA_API gnna_status gnna_features_close(gnna_ctx* ctx, int dtype, const void* d_a, const void* d_b,
                                uint64_t count, double rel_tol, int* close);

/* engine.hpp:66 aggregate_oracle: y[v] = sum in CSR order (K4). */
GNNA_API gnna_status gnna_aggregate_rows(gnna_ctx* ctx, int dtype, const uint64_t* d_row_ptr,
                                const uint32_t* d_col, uint32_t n, uint32_t dim,
                                const void* d_x, void* d_y);

/* Host-buffer entry (what a drop-in aggregate_scheduled call does end to
 * end): uploads CSR + x, plans, aggregates, downloads y (and the cost report
 * when cost != NULL).  Host buffers may be pageable or pinned. */
GNNA_API gnna_status gnna_aggregate_host(gnna_ctx* ctx, int dtype, const uint64_t* h_row_ptr,
                                const uint32_t* h_col, uint32_t n, const gnna_params* p,
                                int strategy, int dim_mode, const void* h_x, void* h_y,
                                uint64_t line_bytes, uint64_t cache_capacity,
                                uint64_t cache_line, gnna_cost* cost);

/* Row-shard variant (multi-GPU row sharding): rows
 * [row_begin, row_end) of the host CSR are aggregated over the full host
 * feature matrix; only the shard's CSR slice is uploaded and h_y receives
 * (row_end - row_begin) x dim values.  The cost report (when requested)
 * describes the shard's own schedule. */
GNNA_API gnna_status gnna_aggregate_host_rows(gnna_ctx* ctx, int dtype, const uint64_t* h_row_ptr,
                                     const uint32_t* h_col, uint32_t n, uint32_t row_begin,
                                     uint32_t row_end, const gnna_params* p, int strategy,
                                     int dim_mode, const void* h_x, void* h_y,
                                     uint64_t line_bytes, uint64_t cache_capacity,
                                     uint64_t cache_line, gnna_cost* cost);

/* A stream of host-buffer aggregations (one per batch: its own CSR row
 * range and features), pipelined: batch i+1's uploads overlap batch i's
 * planning + K3 and batch i-1's download (two device buffer sets, separate
 * copy streams; PCIe is full duplex).  Same results as calling
 * gnna_aggregate_host_rows per batch.  Host buffers should be pinned. */
typedef struct {
    const uint64_t* h_row_ptr;
    const uint32_t* h_col;
    uint32_t n, row_begin, row_end;
    const void* h_x;
    void* h_y;  /* (row_end - row_begin) x dim */
} gnna_host_batch;
GNNA_API gnna_status gnna_aggregate_host_stream(gnna_ctx* ctx, int dtype, const gnna_params* p, int strategy,
                                       int dim_mode, const gnna_host_batch* batches,
                                       uint32_t num_batches);

/* -------------------------------------------------------- GCN / GIN --- */
/* engine.cpp:340-353: norm[v] = 1/sqrt(max(deg'(v),1)) (f64), deg' counts an
 * implicit self loop when add_self_loops and v has none; d_self (u8, may be
 * NULL) receives the implicit-self flags. */
GNNA_API gnna_status gnna_gcn_norm(gnna_ctx* ctx, const uint64_t* d_row_ptr, const uint32_t* d_col,
                          uint32_t n, int add_self_loops, double* d_norm, uint8_t* d_self);
/* fp32 operands of the fused normalized aggregation (gnna_aggregate_ex):
 * d_row_scale[v] = norm[v], d_self_weight[v] = norm[v] if v gets an implicit
 * self loop else 0, d_edge_weight[e] = norm[col[e]] (any may be NULL).  With
 * node_weight = row_scale (= norm), gnna_aggregate_ex computes
 * y = row_scale * (A (norm x) + self_weight * x) = D^-1/2 (A [+I]) D^-1/2 x. */
GNNA_API gnna_status gnna_gcn_weights(gnna_ctx* ctx, const uint64_t* d_row_ptr, const uint32_t* d_col,
                             uint32_t n, int add_self_loops, float* d_row_scale,
                             float* d_self_weight, float* d_edge_weight);
/* Operands of the FOLDED normalisation (the GCN layer's fast form): when the
 * aggregation's input comes from the update GEMM, the source-side D^-1/2 rides
 * in the GEMM's row-scale epilogue (gnna_gemm epilogue 2 with d_norm), so the
 * aggregation is a plain sum:
 *   y = row_scale * (A t' + self_ind * t'),  t' = norm * (X W)
 * d_norm[v] (f64) = norm[v] (the GEMM epilogue's row scale); d_row_scale[v] =
 * norm[v]; d_row_scale2[v] = norm[v]^2 (an aggregation whose output feeds the
 * next aggregation directly: its epilogue pre-scales it); d_self_ind[v] = 1 if
 * v gets an implicit self loop else 0.  Any output may be NULL. */
GNNA_API gnna_status gnna_gcn_fold_weights(gnna_ctx* ctx, const uint64_t* d_row_ptr, const uint32_t* d_col,
                                           uint32_t n, int add_self_loops, double* d_norm, float* d_row_scale,
                                           float* d_row_scale2, float* d_self_ind);
/* engine.cpp:338-369 normalized_aggregate, z = D^-1/2 (A [+I]) D^-1/2 x,
 * F64 bitwise as the reference.  transpose != 0 applies the adjoint
 * (out[u] += norm[v]norm[u] x[v]); it requires the transposed CSR
 * (gnna_csr_transpose), which for a symmetric CSR is the CSR itself. */
GNNA_API gnna_status gnna_normalized_aggregate(gnna_ctx* ctx, int dtype, const uint64_t* d_row_ptr,
                                      const uint32_t* d_col, uint32_t n, uint32_t dim,
                                      const double* d_norm, const uint8_t* d_self,
                                      const void* d_x, void* d_y);
/* engine.cpp:315-331 matmul (K6): out = a (m x k) . w (k x n_out) [+ bias]
 * [relu].  F64: k ascending, a==0 skipped, separate multiply and add —
 * bitwise equal to the reference.  epilogue: 0 none, 1 bias+relu (GIN),
 * 2 row scale by d_row_scale (f64 vector, used by the fp32 GCN fold). */
GNNA_API gnna_status gnna_gemm(gnna_ctx* ctx, int dtype, const void* d_a, uint32_t m, uint32_t k,
                      const void* d_w, uint32_t n_out, const void* d_bias, int epilogue,
                      const double* d_row_scale, void* d_out);
/* Weight gradient product out (p x q) = a^T b, a: m x p, b: m x q (backward
 * of matmul; row-chunk partials summed in chunk order: deterministic). */
GNNA_API gnna_status gnna_gemm_tn(gnna_ctx* ctx, int dtype, const void* d_a, const void* d_b, uint32_t m,
                         uint32_t p, uint32_t q, void* d_out);
/* Backward of the node update y = z W (matmul, engine.cpp:315-331; no
 * reference backward exists): dz (m x p) = row_scale ⊙ (dy Wᵀ)
 * (row_scale may be null) and dW (p x q) = zᵀ dy, for dy (m x q), W (p x q),
 * z (m x p).  F32 with p, q <= 32 runs ONE fused pass over the rows (the
 * narrow GCN output layer); otherwise the two products run separately
 * (F64: the exact orders of gnna_gemm / gnna_gemm_tn). */
GNNA_API gnna_status gnna_dense_backward(gnna_ctx* ctx, int dtype, const void* d_dy, uint32_t m, uint32_t q,
                                const void* d_w, const void* d_z, uint32_t p, const double* d_row_scale,
                                void* d_dz, void* d_dw);
/* engine.hpp:93 gcn_layer / engine.hpp:108 gin_layer, forward (F64 bitwise;
 * F32 runs a scheduled plan with the normalisation fused into K3). */
GNNA_API gnna_status gnna_gcn_forward(gnna_ctx* ctx, int dtype, const uint64_t* d_row_ptr,
                             const uint32_t* d_col, uint32_t n, const void* d_x,
                             uint32_t in_dim, const void* d_w, uint32_t out_dim,
                             int add_self_loops, void* d_y);
GNNA_API gnna_status gnna_gin_forward(gnna_ctx* ctx, int dtype, const uint64_t* d_row_ptr,
                             const uint32_t* d_col, uint32_t n, const void* d_x,
                             uint32_t in_dim, double eps, const void* d_w, uint32_t out_dim,
                             const void* d_b, void* d_y);
/* Backward entry points (no reference function: SPEC.md:9 lists autograd as
 * out of scope; added in the same style).  d_rt_ptr/d_rt_col is the
 * transposed CSR (pass the CSR itself when it is symmetric, as to_csr(...,
 * true) produces).  Gradients: GCN dx, dw; GIN dx, dw, db, deps (host). */
GNNA_API gnna_status gnna_gcn_backward(gnna_ctx* ctx, int dtype, const uint64_t* d_row_ptr,
                              const uint32_t* d_col, const uint64_t* d_rt_ptr,
                              const uint32_t* d_rt_col, uint32_t n, const void* d_x,
                              uint32_t in_dim, const void* d_w, uint32_t out_dim,
                              int add_self_loops, const void* d_dy, void* d_dx, void* d_dw);
GNNA_API gnna_status gnna_gin_backward(gnna_ctx* ctx, int dtype, const uint64_t* d_row_ptr,
                              const uint32_t* d_col, const uint64_t* d_rt_ptr,
                              const uint32_t* d_rt_col, uint32_t n, const void* d_x,
                              uint32_t in_dim, double eps, const void* d_w, uint32_t out_dim,
                              const void* d_b, const void* d_dy, void* d_dx, void* d_dw,
                              void* d_db, double* deps);

/* -------------------------------------------------- graph utilities --- */
/* graph.cpp:76 to_csr on the GPU (symmetrize, sort rows, drop duplicates).
 * Two-phase: call with d_col == NULL to get *nnz, then with a buffer of
 * *nnz entries.  d_edges: E (src,dst) u32 pairs. */
GNNA_API gnna_status gnna_to_csr(gnna_ctx* ctx, uint32_t n, const uint32_t* d_edges, uint64_t e,
                        int symmetrize, uint64_t* d_row_ptr, uint32_t* d_col, uint64_t* nnz);
/* CSR transpose (for the backward of non-symmetric graphs). */
GNNA_API gnna_status gnna_csr_transpose(gnna_ctx* ctx, const uint64_t* d_row_ptr, const uint32_t* d_col,
                               uint32_t n, uint64_t* d_t_ptr, uint32_t* d_t_col);
/* graph.cpp:122 aes (exact u64 span sum, then one divide). */
GNNA_API gnna_status gnna_aes(gnna_ctx* ctx, const uint32_t* d_edges, uint64_t e, double* out);
/* graph.cpp:106 degree_stats */
GNNA_API gnna_status gnna_degree_stats(gnna_ctx* ctx, const uint64_t* d_row_ptr, uint32_t n, double* avg,
                              uint64_t* max_degree, double* stddev);

/* -------------------------------------------------------- renumbering --- */
/* renumber.cpp:31 detect_communities (exact greedy modularity merge order). */
GNNA_API gnna_status gnna_detect_communities(gnna_ctx* ctx, const uint64_t* d_row_ptr,
                                    const uint32_t* d_col, uint32_t n, uint32_t* d_com,
                                    uint32_t* num_communities);
/* renumber.cpp:106 modularity */
GNNA_API gnna_status gnna_modularity(gnna_ctx* ctx, const uint64_t* d_row_ptr, const uint32_t* d_col,
                            uint32_t n, const uint32_t* d_com, uint32_t num_communities,
                            double* q);
/* renumber.cpp:128 build_mapping: order by (community, old id). */
GNNA_API gnna_status gnna_build_mapping(gnna_ctx* ctx, const uint32_t* d_com, uint32_t n,
                               uint32_t num_communities, uint32_t* d_old_to_new,
                               uint32_t* d_new_to_old);
/* Degree order (B200 addition, no reference counterpart): new ids by
 * descending degree, ties by old id.  Numbering the power-law hubs first
 * makes them one contiguous front block of the feature matrix, which
 * gnna_set_l2_window can keep resident in L2.  Apply with
 * gnna_apply_mapping_csr and a row gather of the features. */
GNNA_API gnna_status gnna_degree_order(gnna_ctx* ctx, const uint64_t* d_row_ptr, uint32_t n,
                                       uint32_t* d_old_to_new, uint32_t* d_new_to_old);
/* renumber.cpp:148 mapping_from_vector (DOMAIN if not a permutation). */
/* ------------------------------------------------- synthetic inputs --- */
/* Host-only (no device needed).  Edge samplers for the BASELINE configs with
 * the reference's generator family (std::mt19937_64 + draw_unit /
 * draw_index, rand.hpp:13-21); out_edges: pairs x 2 node ids.  Pairs are
 * drawn in fixed chunks of 2^20 (chunk c from mt19937_64(seed + c *
 * 0x9E3779B97F4A7C15)) on all host threads: output independent of the thread
 * count.  shuffle: ids permuted by Fisher-Yates with draw_index (the
 * planted_partition shuffle, pipeline.cpp:37-44).
 * Chung-Lu: endpoint weight (i + i0)^-(1/(gamma-1)), inverse-CDF sampling.
 * SBM: equal contiguous blocks; an endpoint stays in its source's block with
 * probability p_intra.  random_features is pipeline.cpp:57-67 exactly (one
 * sequential stream, row-major U[0,1)); the F32 form casts the same doubles. */
GNNA_API gnna_status gnna_gen_chung_lu(uint32_t n, uint64_t pairs, double gamma, double i0, uint64_t seed,
                              int shuffle, uint32_t* out_edges);
GNNA_API gnna_status gnna_gen_sbm(uint32_t n, uint64_t pairs, uint32_t communities, double p_intra,
                         uint64_t seed, int shuffle, uint32_t* out_edges);
GNNA_API gnna_status gnna_random_features(uint32_t n, uint32_t dim, uint64_t seed, int dtype, void* out);

/* Hub rows kept in L2 WITHOUT renumbering (drop-in path: the caller's node
 * order, and so the reference's summation tree, stay as they are).  Picks
 * the k highest-degree nodes (ties by id: the gnna_degree_order keys) into
 * d_hubs[k] and writes d_col_out = d_col with every entry that names a hub
 * replaced by n + its hub slot; *hub_edges = entries replaced (the hubs'
 * gather share).  A plan built over d_col_out reads a hub's row from rows
 * [n, n + k) of an extended feature buffer whose tail holds copies of the
 * hub rows (gnna_gather_rows): the same values in the same order, so the
 * result is bit-identical, while the hot rows are one contiguous block that
 * gnna_set_l2_window can pin (the reference renumbers for locality,
 * renumber.cpp; this keeps its order and gets B200's L2). */
GNNA_API gnna_status gnna_hub_remap(gnna_ctx* ctx, const uint64_t* d_row_ptr, const uint32_t* d_col, uint32_t n,
                           uint32_t k, uint32_t* d_hubs, uint32_t* d_col_out, uint64_t* hub_edges);
/* d_out[i][:] = d_x[d_rows[i]][:] for i < count. */
GNNA_API gnna_status gnna_gather_rows(gnna_ctx* ctx, int dtype, const void* d_x, uint32_t dim,
                             const uint32_t* d_rows, uint64_t count, void* d_out);
GNNA_API gnna_status gnna_mapping_from_vector(gnna_ctx* ctx, const uint32_t* d_vec, uint32_t n,
                                     uint32_t* d_old_to_new, uint32_t* d_new_to_old);
/* renumber.cpp:162 apply_mapping (CSR), output canonical (rows sorted). */
GNNA_API gnna_status gnna_apply_mapping_csr(gnna_ctx* ctx, const uint64_t* d_row_ptr,
                                   const uint32_t* d_col, uint32_t n,
                                   const uint32_t* d_old_to_new, const uint32_t* d_new_to_old,
                                   uint64_t* d_out_row_ptr, uint32_t* d_out_col);
/* renumber.cpp:187 apply_mapping (EdgeList). */
GNNA_API gnna_status gnna_apply_mapping_edges(gnna_ctx* ctx, const uint32_t* d_edges, uint64_t e,
                                     uint32_t n, const uint32_t* d_old_to_new,
                                     uint32_t* d_out_edges);

/* ------------------------------------- performance evaluator (host) --- */
/* decider.hpp:46-94, the reference's model with its defaults. */
GNNA_API gnna_status gnna_model_inputs_from_graph(gnna_ctx* ctx, const uint64_t* d_row_ptr, uint32_t n,
                                         uint32_t dim, gnna_model_inputs* out);
/* Message of the last evaluator DomainError on this thread (decider.cpp's text). */
GNNA_API const char* gnna_decider_last_error(void);
GNNA_API double gnna_alpha_from_degrees(double avg_degree, double stddev_degree);
GNNA_API gnna_status gnna_select_dw(uint32_t dim, uint32_t tpw, uint32_t* out);
GNNA_API gnna_status gnna_select_ngs(uint32_t dw, uint32_t tpb, const gnna_model_inputs* in,
                            uint32_t* out);
GNNA_API gnna_status gnna_dp_size(uint64_t smem_bytes, double avg_degree, double* out);
GNNA_API gnna_status gnna_estimate_latency(const gnna_params* p, const gnna_model_inputs* in,
                                  double* out);
GNNA_API int gnna_candidate_feasible(const gnna_params* p, const gnna_model_inputs* in);
GNNA_API int gnna_feasibility(const gnna_params* p, const gnna_model_inputs* in);
GNNA_API gnna_status gnna_auto_params(const gnna_model_inputs* in, gnna_params* out);
GNNA_API gnna_status gnna_search_params(const gnna_model_inputs* in, uint32_t iterations,
                               uint32_t population, uint64_t seed, const uint32_t* gs_values,
                               uint32_t n_gs, const uint32_t* dw_values, uint32_t n_dw,
                               const uint32_t* tpb_values, uint32_t n_tpb, gnna_params* best,
                               double* est_latency, int* feasible, double* trace,
                               uint32_t* trace_len);
/* B200 profile of the evaluator: 148 SMs, 227 KiB smem per block, runtime
 * L2/HBM figures.  Fills `in` device fields from the live device. */
GNNA_API gnna_status gnna_b200_profile(gnna_ctx* ctx, gnna_model_inputs* in);
/* B200 evaluator (north-star subsystem 3): picks ngs from a calibrated
 * cost model T(ngs) = max(B_alg/BW + G(ngs)*c_unit,
 *                         c_ramp*B_alg/BW + min(ngs, max_degree)*c_edge)
 * with G = n + nnz/ngs (c_unit 24 ps, c_edge 95 ns, c_ramp 0.46, fitted on
 * measured K3 sweeps); tpb = 512; dw = select_dw(dim).  hbm_gbs <= 0 uses
 * 6553 (MEASURED_PEAKS.json).  *est_us (may be NULL) = the model's K3 time. */
/* The B200 evaluator on a device graph: reads the degree profile (max
 * degree; the gather share of the highest-degree rows that fit in half the
 * L2 and in a 48 MB window) and the device's SM count and L2 size, and
 * returns the parameters (ngs; tpb 512; dw = select_dw), the model's K3
 * estimate (us) and the recommended L2 window for the hub rows (0: none).
 * hbm_gbs <= 0: the B200's measured 6,544.7 GB/s.  dtype: element size. */
GNNA_API gnna_status gnna_b200_plan_params(gnna_ctx* ctx, const uint64_t* d_row_ptr, uint32_t n, uint32_t dim,
                                  int dtype, double hbm_gbs, gnna_params* out, double* est_us,
                                  uint64_t* l2_window_bytes);
GNNA_API gnna_status gnna_b200_auto_params(const gnna_model_inputs* in, uint64_t max_degree, double hbm_gbs,
                                  gnna_params* out, double* est_us);
/* Measured-latency tuner: times gnna_aggregate (F32) on the live graph for
 * every (ngs, dw, tpb) in the grid and returns the fastest (K3 sweep). */
GNNA_API gnna_status gnna_tune_params(gnna_ctx* ctx, const uint64_t* d_row_ptr, const uint32_t* d_col,
                             uint32_t n, uint32_t dim, const uint32_t* gs_values, uint32_t n_gs,
                             const uint32_t* dw_values, uint32_t n_dw,
                             const uint32_t* tpb_values, uint32_t n_tpb, gnna_params* best,
                             float* best_ms);

#ifdef __cplusplus
}
#endif
#endif /* GNNA_H */
