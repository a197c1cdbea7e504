// K8: the integer CostReport of aggregate_scheduled (engine.cpp:242-297) and
// the per-block LRU replay (engine.cpp:51-101, simulate_cache), on the GPU.
//
// Counters use closed forms (verified against oracle/_ref in tests/):
//   global_reads  = nnz * dim
//   atomic_ops = global_writes = nnz*dim (Naive) | G*dim (UnitSync) | leaders*dim (WarpShared)
//   global_transactions = sum_e L(col[e]) + {Naive: sum_e L(target(e)),
//                         UnitSync: sum_units L(target), WarpShared: sum_leaders L(node)}
// where L(u) = sum_iter step_lines(u*dim*4, iter) depends on (u*dim*4) mod
// line only, so it is tabulated once per (dim, dw, mode, line).
// The LRU replay is sequential inside a schedule block but blocks are
// independent: one warp per block, lanes search the resident lines in
// parallel, recency is a per-block clock (evict = minimum stamp).
#include <algorithm>
#include <cstring>

#include "gnna_common.cuh"

namespace {

using gnna::DevBuf;

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

struct LaneMap {
    uint32_t dim, dw, iters, chunk;
    int seq;
    // dimension handled by lane t at step iter, or -1 (partition_dims, schedule.cpp:32-47)
    __device__ __forceinline__ int64_t at(uint32_t t, uint32_t iter) const {
        if (seq) {
            const uint64_t d = (uint64_t)t * chunk + iter;
            return (iter < chunk && d < dim) ? (int64_t)d : -1;
        }
        const uint64_t d = (uint64_t)t + (uint64_t)iter * dw;
        return d < dim ? (int64_t)d : -1;
    }
};

// engine.cpp:36-49 step_lines summed over all iterations for a row base.
__device__ uint64_t row_lines(uint64_t base, const LaneMap& m, uint64_t line) {
    uint64_t total = 0;
    for (uint32_t it = 0; it < m.iters; ++it) {
        uint64_t prev = ~0ull;
        for (uint32_t t = 0; t < m.dw; ++t) {
            const int64_t d = m.at(t, it);
            if (d < 0) continue;
            const uint64_t l = (base + (uint64_t)d * 4) / line;
            if (l != prev) {
                ++total;
                prev = l;
            }
        }
    }
    return total;
}

__global__ void k8_table(LaneMap m, uint64_t line, uint32_t* __restrict__ table) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < line; r += (uint64_t)gridDim.x * blockDim.x)
        table[r] = (uint32_t)row_lines(r, m, line);
}

struct CountArgs {
    const uint64_t* part_ptr;
    const uint32_t* part2node;
    const uint8_t* leader;
    const uint32_t* col;
    uint64_t G;
    uint32_t dim;
    uint64_t line;
    const uint32_t* table;  // null -> direct evaluation
    LaneMap m;
    int strategy;
};

__device__ __forceinline__ uint64_t L_of(const CountArgs& a, uint32_t u) {
    const uint64_t base = (uint64_t)u * a.dim * 4;
    return a.table ? a.table[base % a.line] : row_lines(base, a.m, a.line);
}

__device__ __forceinline__ uint64_t warp_sum(uint64_t v) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// out[0] = transactions, out[1] = leaders
__global__ void k8_count(CountArgs a, unsigned long long* __restrict__ out) {
    uint64_t tx = 0, leaders = 0;
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < a.G; u += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = a.part_ptr[u], e = a.part_ptr[u + 1];
        const uint32_t t = a.part2node[u];
        for (uint64_t p = b; p < e; ++p) tx += L_of(a, a.col[p]);
        if (a.strategy == GNNA_NAIVE_ATOMIC) {
            tx += (e - b) * L_of(a, t);
        } else if (a.strategy == GNNA_UNIT_SYNC) {
            tx += L_of(a, t);
        } else if (a.leader[u]) {
            tx += L_of(a, t);
        }
        leaders += a.leader[u] ? 1 : 0;
    }
    tx = warp_sum(tx);
    leaders = warp_sum(leaders);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&out[0], (unsigned long long)tx);
        atomicAdd(&out[1], (unsigned long long)leaders);
    }
}

// ---------------------------------------------------------- LRU replay ---
struct ReplayArgs {
    const uint64_t* begin;  // per warp CSR range [begin[w], end[w])
    const uint64_t* end;
    const uint32_t* col;
    uint64_t G;
    uint32_t wpb;
    uint64_t row_bytes;
    uint64_t line;
    uint64_t cap;   // lines
    uint32_t ecap;  // entries per warp in the scratch table
};

__device__ __forceinline__ uint64_t nlines(uint64_t u, const ReplayArgs& a) {
    const uint64_t base = u * a.row_bytes;
    return (base + a.row_bytes - 1) / a.line - base / a.line + 1;
}

// Upper bound of distinct lines per block: its access count.
__global__ void k8_block_access(ReplayArgs a, unsigned long long* __restrict__ maxacc) {
    const uint64_t nblk = (a.G + a.wpb - 1) / a.wpb;
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t sb = blockIdx.x * (uint64_t)(blockDim.x / 32) + threadIdx.x / 32; sb < nblk;
         sb += (uint64_t)gridDim.x * (blockDim.x / 32)) {
        uint64_t acc = 0;
        for (uint64_t w = sb * a.wpb; w < umin64((sb + 1) * a.wpb, a.G); ++w)
            for (uint64_t p = a.begin[w] + lane; p < a.end[w]; p += 32) acc += nlines(a.col[p], a);
        acc = warp_sum(acc);
        if (lane == 0) atomicMax(maxacc, (unsigned long long)acc);
    }
}

template <bool SMEM>
__global__ void k8_replay(ReplayArgs a, uint64_t* __restrict__ gkeys, uint32_t* __restrict__ gstamp,
                          unsigned long long* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x / 32;
    const uint64_t gw = blockIdx.x * (uint64_t)(blockDim.x / 32) + wib;
    uint64_t* keys;
    uint32_t* stamp;
    if (SMEM) {
        keys = reinterpret_cast<uint64_t*>(smem_raw) + (size_t)wib * a.ecap;
        stamp = reinterpret_cast<uint32_t*>(reinterpret_cast<uint64_t*>(smem_raw) + (size_t)(blockDim.x / 32) * a.ecap) +
                (size_t)wib * a.ecap;
    } else {
        keys = gkeys + gw * a.ecap;
        stamp = gstamp + gw * a.ecap;
    }
    const uint64_t nblk = (a.G + a.wpb - 1) / a.wpb;
    uint64_t hits = 0, accesses = 0;
    for (uint64_t sb = gw; sb < nblk; sb += (uint64_t)gridDim.x * (blockDim.x / 32)) {
        const uint64_t u0 = sb * a.wpb;
        const uint32_t nw = (uint32_t)umin64(a.wpb, a.G - u0);
        uint64_t myb = 0, mysz = 0;
        if (lane < nw) {
            myb = a.begin[u0 + lane];
            mysz = a.end[u0 + lane] - myb;
        }
        uint64_t maxsz = mysz;
        for (int o = 16; o; o >>= 1) maxsz = max(maxsz, __shfl_xor_sync(0xffffffffu, maxsz, o));
        uint32_t size = 0, clock = 0;
        for (uint64_t k = 0; k < maxsz; ++k) {
            for (uint32_t w = 0; w < nw; ++w) {
                const uint64_t bw = __shfl_sync(0xffffffffu, myb, w);
                const uint64_t sw = __shfl_sync(0xffffffffu, mysz, w);
                if (k >= sw) continue;
                const uint64_t base = (uint64_t)a.col[bw + k] * a.row_bytes;
                const uint64_t first = base / a.line, last = (base + a.row_bytes - 1) / a.line;
                for (uint64_t l = first; l <= last; ++l) {
                    ++accesses;
                    ++clock;
                    int found = -1;
                    for (uint32_t i = lane; i < size; i += 32)
                        if (keys[i] == l) found = (int)i;
                    const uint32_t fm = __ballot_sync(0xffffffffu, found >= 0);
                    if (fm) {
                        ++hits;
                        if (lane == __ffs(fm) - 1) stamp[found] = clock;
                    } else if (size < a.cap) {
                        if (lane == 0) {
                            keys[size] = l;
                            stamp[size] = clock;
                        }
                        ++size;
                    } else {
                        // evict the least recently used entry (minimum stamp)
                        uint32_t best = 0xffffffffu, bi = 0;
                        for (uint32_t i = lane; i < size; i += 32)
                            if (stamp[i] < best) {
                                best = stamp[i];
                                bi = i;
                            }
                        for (int o = 16; o; o >>= 1) {
                            const uint32_t ob = __shfl_xor_sync(0xffffffffu, best, o);
                            const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
                            if (ob < best || (ob == best && oi < bi)) {
                                best = ob;
                                bi = oi;
                            }
                        }
                        __syncwarp();  // all lanes' stamp reads above precede lane 0's overwrite (WAR)
                        if (lane == 0) {
                            keys[bi] = l;
                            stamp[bi] = clock;
                        }
                    }
                    __syncwarp();
                }
            }
        }
    }
    if (lane == 0) {
        atomicAdd(&out[0], (unsigned long long)hits);
        atomicAdd(&out[1], (unsigned long long)accesses);
    }
}

void cache_validate(uint64_t cap, uint64_t line) {
    // engine.cpp:141-145 CacheConfig::validate
    if (line == 0) gnna::raise(GNNA_ERR_DOMAIN, "cache line size must be positive");
    if (cap < line || cap % line != 0)
        gnna::raise(GNNA_ERR_DOMAIN, "cache capacity must be a positive multiple of the line size");
}

void replay_ranges(gnna_ctx* ctx, const uint64_t* begin, const uint64_t* end, const uint32_t* col, uint64_t G,
                   uint32_t wpb, uint64_t cap_bytes, uint64_t line, uint32_t dim, uint64_t* hits, uint64_t* accesses) {
    cudaStream_t s = ctx->stream;
    *hits = *accesses = 0;
    if (G == 0) return;
    ReplayArgs a{};
    a.begin = begin;
    a.end = end;
    a.col = col;
    a.G = G;
    a.wpb = wpb;
    a.row_bytes = (uint64_t)dim * 4;
    a.line = line;
    a.cap = cap_bytes / line;
    DevBuf<unsigned long long> mx(1, s);
    GNNA_CUDA(cudaMemsetAsync(mx.get(), 0, 8, s));
    const uint64_t nblk = (a.G + a.wpb - 1) / a.wpb;
    k8_block_access<<<gnna::grid_for(nblk * 32, 256, 1 << 16), 256, 0, s>>>(a, mx.get());
    gnna::launched(ctx, "k8_block_access");
    unsigned long long maxacc = 0;
    gnna::to_host(ctx, &maxacc, mx.get(), 1);
    const uint64_t ecap = std::min<uint64_t>(a.cap, maxacc);
    if (ecap == 0) return;
    if (ecap > (1ull << 31)) gnna::raise(GNNA_ERR_DOMAIN, "cache replay: block too large");
    a.ecap = (uint32_t)ecap;
    DevBuf<unsigned long long> out(2, s);
    GNNA_CUDA(cudaMemsetAsync(out.get(), 0, 16, s));
    const int warps = 4;
    const size_t smem = (size_t)warps * ecap * 12;
    if (smem <= 200 * 1024) {
        if (smem > 48 * 1024)
            GNNA_CUDA(cudaFuncSetAttribute(k8_replay<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const unsigned grid = (unsigned)std::min<uint64_t>((nblk + warps - 1) / warps, 1u << 20);
        k8_replay<true><<<grid, warps * 32, smem, s>>>(a, nullptr, nullptr, out.get());
    } else {
        const unsigned grid = (unsigned)std::min<uint64_t>((nblk + warps - 1) / warps, (uint64_t)ctx->num_sms * 8);
        DevBuf<uint64_t> keys((uint64_t)grid * warps * ecap, s);
        DevBuf<uint32_t> st((uint64_t)grid * warps * ecap, s);
        k8_replay<false><<<grid, warps * 32, 0, s>>>(a, keys.get(), st.get(), out.get());
    }
    gnna::launched(ctx, "k8_replay");
    unsigned long long r[2];
    gnna::to_host(ctx, r, out.get(), 2);
    *hits = r[0];
    *accesses = r[1];
}

void replay(gnna_ctx* ctx, const gnna_plan* plan, uint64_t cap_bytes, uint64_t line, uint32_t dim, uint64_t* hits,
            uint64_t* accesses) {
    replay_ranges(ctx, plan->part_ptr.get(), plan->part_ptr.get() + 1, plan->col, plan->G, plan->wpb_params, cap_bytes,
                  line, dim, hits, accesses);
}

}  // namespace

namespace gnna {

void cost_report(gnna_ctx* ctx, const gnna_plan* plan, int dim_mode, uint64_t line, uint64_t cache_cap,
                 uint64_t cache_line, gnna_cost* out) {
    if (!plan) raise(GNNA_ERR_DOMAIN, "null plan");
    if (line == 0) raise(GNNA_ERR_DOMAIN, "transaction line size must be positive");
    if (cache_line) cache_validate(cache_cap, cache_line);
    cudaStream_t s = ctx->stream;
    const gnna_params& p = plan->params;
    const uint32_t dim = p.dim;
    std::memset(out, 0, sizeof(*out));
    uint64_t nnz_lo = 0, nnz_hi = 0;
    to_host(ctx, &nnz_lo, plan->row_ptr + plan->row_begin, 1);
    to_host(ctx, &nnz_hi, plan->row_ptr + plan->row_end, 1);
    const uint64_t nnz = nnz_hi - nnz_lo;
    out->global_reads = nnz * dim;
    LaneMap m{dim, p.dw, (dim + p.dw - 1) / p.dw, (dim + p.dw - 1) / p.dw, dim_mode == GNNA_DIM_SEQUENTIAL};
    DevBuf<uint32_t> table;
    if (line <= (1u << 16)) {
        table = DevBuf<uint32_t>(line, s);
        k8_table<<<grid_for(line, 128), 128, 0, s>>>(m, line, table.get());
        launched(ctx, "k8_table");
    }
    uint64_t tx = 0, leaders = 0;
    if (plan->G) {
        CountArgs a{plan->part_ptr.get(), plan->part2node.get(), plan->leader.get(), plan->col, plan->G, dim, line,
                    table.get(), m, plan->strategy};
        DevBuf<unsigned long long> acc(2, s);
        GNNA_CUDA(cudaMemsetAsync(acc.get(), 0, 16, s));
        k8_count<<<grid_for(plan->G, 256, (uint64_t)ctx->num_sms * 16), 256, 0, s>>>(a, acc.get());
        launched(ctx, "k8_count");
        unsigned long long r[2];
        to_host(ctx, r, acc.get(), 2);
        tx = r[0];
        leaders = r[1];
    }
    out->global_transactions = tx;
    switch (plan->strategy) {
        case GNNA_NAIVE_ATOMIC:
            out->atomic_ops = out->global_writes = nnz * dim;
            break;
        case GNNA_UNIT_SYNC:
            out->atomic_ops = out->global_writes = plan->G * dim;
            break;
        default:
            out->atomic_ops = out->global_writes = leaders * dim;
            out->shared_bytes_per_block = (uint64_t)plan->wpb_params * dim * 4;
    }
    if (cache_line) replay(ctx, plan, cache_cap, cache_line, dim, &out->cache_hits, &out->cache_accesses);
}

}  // namespace gnna

extern "C" {

gnna_status gnna_cost_report(gnna_ctx* ctx, const gnna_plan* plan, int dim_mode, uint64_t line_bytes,
                             uint64_t cache_capacity, uint64_t cache_line, gnna_cost* out) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        gnna::cost_report(ctx, plan, dim_mode, line_bytes, cache_capacity, cache_line, out);
    });
}

gnna_status gnna_simulate_cache(gnna_ctx* ctx, const gnna_plan* plan, uint64_t cache_capacity, uint64_t cache_line,
                                uint32_t dim, uint64_t* hits, uint64_t* accesses) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (!plan) gnna::raise(GNNA_ERR_DOMAIN, "null plan");
        cache_validate(cache_capacity, cache_line);
        if (dim == 0) gnna::raise(GNNA_ERR_DOMAIN, "dim must be positive");
        replay(ctx, plan, cache_capacity, cache_line, dim, hits, accesses);
    });
}

gnna_status gnna_simulate_cache_ranges(gnna_ctx* ctx, const uint32_t* d_col, const uint64_t* d_begin,
                                       const uint64_t* d_end, uint64_t num_warps, uint32_t warps_per_block,
                                       uint64_t cache_capacity, uint64_t cache_line, uint32_t dim, uint64_t* hits,
                                       uint64_t* accesses) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        cache_validate(cache_capacity, cache_line);
        if (dim == 0) gnna::raise(GNNA_ERR_DOMAIN, "dim must be positive");
        if (warps_per_block < 1 || warps_per_block > 32) gnna::raise(GNNA_ERR_DOMAIN, "warps per block must be in [1, 32]");
        replay_ranges(ctx, d_begin, d_end, d_col, num_warps, warps_per_block, cache_capacity, cache_line, dim, hits,
                      accesses);
    });
}

}  // extern "C"
