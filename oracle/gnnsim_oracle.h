/* TEST INFRASTRUCTURE ONLY — the CPU parity oracle.  Never linked into the
 * product (paper_2006_06608_b200/); only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it, and only as the checker.
 *
 * A plain-C restatement of the reference gnnsim aggregation path
 * (/root/reference/proj/src/ sources).  Every entry point mirrors the POD
 * signature of the matching ref_* function in oracle/ref_shim.cpp (the
 * reference itself, compiled from its sources into oracle/_ref/), so a test
 * can run the same case through both and through the CUDA C-ABI.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement against the
 * reference's golden vectors (tests/golden/, transcribed from
 * proj/tests/ cases and generated from oracle/_ref by tests/golden/make_golden.py)
 * and differentially against oracle/_ref on seeded corpora.
 *
 * Status codes as ref_shim.cpp: 0 ok, 1 DomainError, 2 InternalError,
 * 6 caller buffer too small.
 */
#ifndef GNNSIM_ORACLE_H
#define GNNSIM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint64_t mt[312];
    int idx;
} orc_rng;

const char* orc_last_error(void);

/* rand.hpp:13-21 + std::mt19937_64 */
void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
uint64_t orc_draw_index(orc_rng* r, uint64_t n);
double orc_draw_unit(orc_rng* r);

int orc_random_features(uint32_t n, uint32_t dim, uint64_t seed, double* out);
int orc_planted_partition(uint32_t communities, uint32_t size, double p_in, double p_out,
                          int shuffle, uint64_t seed, uint64_t cap, uint32_t* edges,
                          uint64_t* num_edges, uint32_t* num_nodes);

int orc_to_csr(uint32_t n, const uint32_t* edges, uint64_t e, int symmetrize,
               uint64_t* row_ptr, uint32_t* col, uint64_t col_cap, uint64_t* nnz);
int orc_aes(uint32_t n, const uint32_t* edges, uint64_t e, double* out);
int orc_should_reorder(uint32_t n, const uint32_t* edges, uint64_t e, int* out);
int orc_degree_stats(uint32_t n, const uint64_t* row_ptr, const uint32_t* col, double* avg,
                     uint64_t* maxd, double* sd);

int orc_validate_params(const uint32_t p[5]);
int orc_partition_neighbors(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                            uint32_t ngs, uint64_t cap, uint64_t* num_groups, uint32_t* ids,
                            uint32_t* targets, uint64_t* begins, uint64_t* ends);
int orc_partition_dims(uint32_t dim, uint32_t dw, int mode, uint32_t* lane_ptr,
                       uint32_t* dims);
int orc_build_mem_plan(const uint32_t* targets, uint64_t num_groups, const uint32_t p[5],
                       uint32_t* slots, uint32_t* nodes, uint8_t* leaders,
                       uint64_t* smem_bytes);

int orc_aggregate_scheduled(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                            const double* x, const uint32_t p[5], int strategy, int dim_mode,
                            uint32_t workers, uint64_t line, int cache_on, uint64_t cache_cap,
                            uint64_t cache_line, double* y, uint64_t cost[7]);
int orc_aggregate_oracle(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                         const double* x, uint32_t dim, double* y);
int orc_count_transactions(const uint64_t* addr, uint64_t k, uint64_t line, uint64_t* out);
int orc_simulate_cache(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                       const uint32_t p[5], uint64_t cache_cap, uint64_t cache_line,
                       uint32_t dim, uint64_t* hits, uint64_t* accesses);

int orc_gcn_layer(uint32_t n, const uint64_t* row_ptr, const uint32_t* col, const double* x,
                  uint32_t in_dim, const double* w, uint32_t out_dim, int self_loops,
                  double* y);
int orc_gin_layer(uint32_t n, const uint64_t* row_ptr, const uint32_t* col, const double* x,
                  uint32_t in_dim, double eps, const double* w, uint32_t out_dim,
                  const double* b, double* y);
/* Backward of gcn_layer / gin_layer.  No reference function exists
 * (SPEC.md:9): these are the analytic gradients of the forward above and are
 * pinned in tests by central finite differences of ref_gcn_layer /
 * ref_gin_layer ("parity unpinned" by the reference itself). */
int orc_gcn_backward(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                     const double* x, uint32_t in_dim, const double* w, uint32_t out_dim,
                     int self_loops, const double* dy, double* dx, double* dw);
int orc_gin_backward(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                     const double* x, uint32_t in_dim, double eps, const double* w,
                     uint32_t out_dim, const double* b, const double* dy, double* dx,
                     double* dw, double* db, double* deps);

int orc_detect_communities(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                           uint32_t* com, uint32_t* ncom);
int orc_modularity(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                   const uint32_t* com, uint32_t ncom, double* q);
int orc_build_mapping(uint32_t n, const uint32_t* com, uint32_t ncom, uint32_t* o2n,
                      uint32_t* n2o);
int orc_mapping_from_vector(uint32_t n, const uint32_t* v, uint32_t* o2n, uint32_t* n2o);
int orc_apply_mapping_csr(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                          const uint32_t* o2n, const uint32_t* n2o, uint64_t* out_row_ptr,
                          uint32_t* out_col);
int orc_apply_mapping_edges(uint32_t n, const uint32_t* edges, uint64_t e,
                            const uint32_t* o2n, const uint32_t* n2o, uint32_t* out);

#ifdef __cplusplus
}
#endif
#endif
