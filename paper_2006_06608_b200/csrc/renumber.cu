// Renumbering on the GPU (renumber.cpp): modularity, build_mapping,
// mapping_from_vector, apply_mapping (CSR and edge list).  All outputs are
// bit-exact with the reference:
//   * build_mapping orders nodes by (community, old id): one LSD radix sort of
//     u64 keys com<<32|id, then a scatter of the ranks;
//   * apply_mapping relabels every edge to new_row<<32|new_col and sorts; rows
//     come out sorted exactly like the reference's per-row std::sort (which
//     keeps duplicates, so no unique pass here);
//   * modularity counts intra/degree per community in u64 (the reference adds
//     1.0 per edge endpoint: exact integers) and sums the per-community terms
//     in ascending community order in one thread, as renumber.cpp:120-124.
// detect_communities (the exact greedy merge) lives in communities.cu.
#include <cub/device/device_select.cuh>

#include "gnna_common.cuh"
#include "host/decider_core.hpp"

namespace gnna {
uint64_t csr_from_keys(gnna_ctx* ctx, uint64_t* keys, uint64_t m, uint32_t n, uint64_t* row_ptr, uint32_t* col,
                       bool dedup);
uint64_t undirected_edges(gnna_ctx* ctx, const uint64_t* row_ptr, const uint32_t* col, uint32_t n,
                          DevBuf<uint64_t>& out);
}  // namespace gnna

namespace {

using gnna::DevBuf;

int bits_for(uint64_t v) {
    int b = 0;
    while (b < 64 && (v >> b)) ++b;
    return b < 1 ? 1 : b;
}

// renumber.cpp:16-27 undirected_edges: {min,max} of every non-loop entry.
__global__ void k7_undirected_keys(const uint64_t* __restrict__ row_ptr, const uint32_t* __restrict__ col, uint32_t n,
                                   uint64_t* __restrict__ keys) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t v = blockIdx.x * (uint64_t)(blockDim.x / 32) + threadIdx.x / 32; v < n; v += warps)
        for (uint64_t p = row_ptr[v] + lane; p < row_ptr[v + 1]; p += 32) {
            const uint32_t u = col[p];
            const uint32_t a = u < v ? u : (uint32_t)v, b = u < v ? (uint32_t)v : u;
            keys[p] = (u == v) ? ~0ull : (((uint64_t)a << 32) | b);
        }
}

__global__ void k7_keep_unique(const uint64_t* __restrict__ k, uint64_t m, uint8_t* __restrict__ keep) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        keep[i] = k[i] != ~0ull && (i == 0 || k[i] != k[i - 1]);
}

__global__ void k7_modularity_counts(const uint64_t* __restrict__ e, uint64_t m, const uint32_t* __restrict__ com,
                                     uint32_t ncom, unsigned long long* __restrict__ deg,
                                     unsigned long long* __restrict__ intra, unsigned* __restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t cu = com[e[i] >> 32], cv = com[(uint32_t)e[i]];
        if (cu >= ncom || cv >= ncom) {
            atomicExch(bad, 1u);
            continue;
        }
        atomicAdd(deg + cu, 1ull);
        atomicAdd(deg + cv, 1ull);
        if (cu == cv) atomicAdd(intra + cu, 1ull);
    }
}

// renumber.cpp:119-124, sequential in community order.
__global__ void k7_modularity_sum(const unsigned long long* __restrict__ deg,
                                  const unsigned long long* __restrict__ intra, uint32_t ncom, double m,
                                  double* __restrict__ q) {
    double s = 0.0;
    const double two_m = __dmul_rn(2.0, m);
    for (uint32_t c = 0; c < ncom; ++c) {
        const double frac = __ddiv_rn((double)deg[c], two_m);
        s = __dadd_rn(s, __dsub_rn(__ddiv_rn((double)intra[c], m), __dmul_rn(frac, frac)));
    }
    *q = s;
}

__global__ void k7_mapping_keys(const uint32_t* __restrict__ com, uint32_t n, uint32_t ncom,
                                uint64_t* __restrict__ keys, unsigned* __restrict__ bad) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        if (com[v] >= ncom) atomicExch(bad, 1u);
        keys[v] = ((uint64_t)com[v] << 32) | v;
    }
}

// Degree order (the L2-residency renumbering): key = (~deg << 32) | id, so an
// ascending sort gives descending degree, ties by id.
__global__ void k7_degree_keys(const uint64_t* __restrict__ row_ptr, uint32_t n, uint64_t* __restrict__ keys) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t d = row_ptr[v + 1] - row_ptr[v];
        const uint32_t dc = d > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)d;
        keys[v] = ((uint64_t)(~dc) << 32) | v;
    }
}

__global__ void k7_mapping_scatter(const uint64_t* __restrict__ keys, uint32_t n, uint32_t* __restrict__ o2n,
                                   uint32_t* __restrict__ n2o) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t old = (uint32_t)keys[i];
        n2o[i] = old;
        o2n[old] = (uint32_t)i;
    }
}

// renumber.cpp:148-160: first (in node order) violation wins the message;
// any violation is reported with the same text.
__global__ void k7_perm_claim(const uint32_t* __restrict__ v2w, uint32_t n, unsigned* __restrict__ owner,
                              unsigned* __restrict__ bad) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t w = v2w[v];
        if (w >= n) {
            atomicExch(bad, 1u);
            continue;
        }
        if (atomicCAS(owner + w, 0xffffffffu, (unsigned)v) != 0xffffffffu) atomicExch(bad, 1u);
    }
}

__global__ void k7_copy_u32(const unsigned* __restrict__ a, uint32_t n, uint32_t* __restrict__ b) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

// apply_mapping (CSR) checks, renumber.cpp:165-169: 1 = size, 2 = not a permutation.
__global__ void k7_check_mapping(const uint32_t* __restrict__ o2n, const uint32_t* __restrict__ n2o, uint32_t n,
                                 unsigned* __restrict__ bad) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x)
        if (o2n[v] >= n || n2o[o2n[v]] != v) atomicExch(bad, 1u);
}

// Relabel: out row o2n[v] gets o2n[u] for every u in N(v).
__global__ void k7_relabel_keys(const uint64_t* __restrict__ row_ptr, const uint32_t* __restrict__ col, uint32_t n,
                                const uint32_t* __restrict__ o2n, uint64_t* __restrict__ keys) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t v = blockIdx.x * (uint64_t)(blockDim.x / 32) + threadIdx.x / 32; v < n; v += warps) {
        const uint64_t nv = o2n[v];
        for (uint64_t p = row_ptr[v] + lane; p < row_ptr[v + 1]; p += 32) keys[p] = (nv << 32) | o2n[col[p]];
    }
}

__global__ void k7_relabel_edges(const uint32_t* __restrict__ e, uint64_t m, uint32_t n,
                                 const uint32_t* __restrict__ o2n, uint32_t* __restrict__ out,
                                 unsigned* __restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint2 uv = reinterpret_cast<const uint2*>(e)[i];
        if (uv.x >= n || uv.y >= n) {
            atomicExch(bad, 1u);
            continue;
        }
        reinterpret_cast<uint2*>(out)[i] = make_uint2(o2n[uv.x], o2n[uv.y]);
    }
}

unsigned read_flag(gnna_ctx* ctx, const DevBuf<unsigned>& f) {
    unsigned h = 0;
    gnna::to_host(ctx, &h, f.get(), 1);
    return h;
}

// Hub rows in L2 without renumbering (gnna_hub_remap / gnna_gather_rows).
__global__ void k7_hub_slots(const uint64_t* __restrict__ sorted_keys, uint32_t k, uint32_t* __restrict__ hubs,
                             uint32_t* __restrict__ slot) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = (uint32_t)(sorted_keys[i] & 0xffffffffu);
        hubs[i] = v;
        slot[v] = (uint32_t)i;
    }
}

__global__ void k7_hub_remap(const uint32_t* __restrict__ col, uint64_t nnz, const uint32_t* __restrict__ slot,
                             uint32_t n, uint32_t* __restrict__ out, unsigned long long* __restrict__ hits) {
    unsigned long long c = 0;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nnz; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t u = col[e], s = slot[u];
        out[e] = s == 0xffffffffu ? u : n + s;
        c += s != 0xffffffffu;
    }
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(hits, c);
}

template <class T>
__global__ void k7_gather_rows(const T* __restrict__ x, uint32_t dim, const uint32_t* __restrict__ rows, uint64_t count,
                               T* __restrict__ out) {
    const uint64_t total = count * dim;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = i / dim, c = i - r * dim;
        out[i] = x[(uint64_t)rows[r] * dim + c];
    }
}

// Sum of the k largest degrees from the sorted (~deg << 32 | id) keys.
__global__ void k7_topk_degree_sum(const uint64_t* __restrict__ keys, uint64_t k, unsigned long long* __restrict__ out) {
    unsigned long long s = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k; i += (uint64_t)gridDim.x * blockDim.x)
        s += (uint32_t)~(uint32_t)(keys[i] >> 32);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

}  // namespace

namespace gnna {

// Sorted unique {min,max} non-loop edges of a CSR (renumber.cpp:16-27).
uint64_t undirected_edges(gnna_ctx* ctx, const uint64_t* row_ptr, const uint32_t* col, uint32_t n,
                          DevBuf<uint64_t>& out) {
    cudaStream_t s = ctx->stream;
    uint64_t nnz = 0;
    to_host(ctx, &nnz, row_ptr + n, 1);
    out = DevBuf<uint64_t>(nnz ? nnz : 1, s);
    if (!nnz) return 0;
    DevBuf<uint64_t> keys(nnz, s);
    k7_undirected_keys<<<grid_for((uint64_t)n * 32, 256), 256, 0, s>>>(row_ptr, col, n, keys.get());
    launched(ctx, "k7_undirected_keys");
    sort_keys_u64(ctx, keys.get(), nnz, 64);
    DevBuf<uint8_t> keep(nnz, s);
    k7_keep_unique<<<grid_for(nnz, 256), 256, 0, s>>>(keys.get(), nnz, keep.get());
    launched(ctx, "k7_keep_unique");
    DevBuf<uint64_t> cnt(1, s);
    size_t bytes = 0;
    GNNA_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, keys.get(), keep.get(), out.get(), cnt.get(), (int64_t)nnz, s));
    DevBuf<uint8_t> tmp(bytes, s);
    GNNA_CUDA(cub::DeviceSelect::Flagged(tmp.get(), bytes, keys.get(), keep.get(), out.get(), cnt.get(), (int64_t)nnz, s));
    uint64_t m = 0;
    to_host(ctx, &m, cnt.get(), 1);
    return m;
}

}  // namespace gnna

extern "C" {

gnna_status gnna_modularity(gnna_ctx* ctx, const uint64_t* d_row_ptr, const uint32_t* d_col, uint32_t n,
                            const uint32_t* d_com, uint32_t num_communities, double* q) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        cudaStream_t s = ctx->stream;
        DevBuf<uint64_t> e;
        const uint64_t m = gnna::undirected_edges(ctx, d_row_ptr, d_col, n, e);
        if (m == 0) {  // renumber.cpp:110
            *q = 0.0;
            return;
        }
        DevBuf<unsigned long long> deg(num_communities ? num_communities : 1, s),
            intra(num_communities ? num_communities : 1, s);
        DevBuf<unsigned> bad(1, s);
        GNNA_CUDA(cudaMemsetAsync(deg.get(), 0, (size_t)(num_communities ? num_communities : 1) * 8, s));
        GNNA_CUDA(cudaMemsetAsync(intra.get(), 0, (size_t)(num_communities ? num_communities : 1) * 8, s));
        GNNA_CUDA(cudaMemsetAsync(bad.get(), 0, 4, s));
        k7_modularity_counts<<<gnna::grid_for(m, 256), 256, 0, s>>>(e.get(), m, d_com, num_communities, deg.get(),
                                                                    intra.get(), bad.get());
        gnna::launched(ctx, "k7_modularity_counts");
        if (read_flag(ctx, bad)) gnna::raise(GNNA_ERR_DOMAIN, "modularity: community index out of range");
        DevBuf<double> out(1, s);
        k7_modularity_sum<<<1, 1, 0, s>>>(deg.get(), intra.get(), num_communities, (double)m, out.get());
        gnna::launched(ctx, "k7_modularity_sum");
        gnna::to_host(ctx, q, out.get(), 1);
    });
}

gnna_status gnna_build_mapping(gnna_ctx* ctx, const uint32_t* d_com, uint32_t n, uint32_t num_communities,
                               uint32_t* d_old_to_new, uint32_t* d_new_to_old) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (!n) return;
        cudaStream_t s = ctx->stream;
        DevBuf<uint64_t> keys(n, s);
        DevBuf<unsigned> bad(1, s);
        GNNA_CUDA(cudaMemsetAsync(bad.get(), 0, 4, s));
        k7_mapping_keys<<<gnna::grid_for(n, 256), 256, 0, s>>>(d_com, n, num_communities, keys.get(), bad.get());
        gnna::launched(ctx, "k7_mapping_keys");
        if (read_flag(ctx, bad)) gnna::raise(GNNA_ERR_DOMAIN, "build_mapping: community index out of range");
        gnna::sort_keys_u64(ctx, keys.get(), n, 32 + bits_for(num_communities ? num_communities - 1 : 0));
        k7_mapping_scatter<<<gnna::grid_for(n, 256), 256, 0, s>>>(keys.get(), n, d_old_to_new, d_new_to_old);
        gnna::launched(ctx, "k7_mapping_scatter");
        GNNA_CUDA(cudaStreamSynchronize(s));
    });
}

gnna_status gnna_degree_order(gnna_ctx* ctx, const uint64_t* d_row_ptr, uint32_t n, uint32_t* d_old_to_new,
                              uint32_t* d_new_to_old) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (!n) return;
        cudaStream_t s = ctx->stream;
        DevBuf<uint64_t> keys(n, s);
        k7_degree_keys<<<gnna::grid_for(n, 256), 256, 0, s>>>(d_row_ptr, n, keys.get());
        gnna::launched(ctx, "k7_degree_keys");
        gnna::sort_keys_u64(ctx, keys.get(), n, 64);
        k7_mapping_scatter<<<gnna::grid_for(n, 256), 256, 0, s>>>(keys.get(), n, d_old_to_new, d_new_to_old);
        gnna::launched(ctx, "k7_mapping_scatter");
    });
}

gnna_status gnna_mapping_from_vector(gnna_ctx* ctx, const uint32_t* d_vec, uint32_t n, uint32_t* d_old_to_new,
                                     uint32_t* d_new_to_old) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (!n) return;
        cudaStream_t s = ctx->stream;
        DevBuf<unsigned> owner(n, s), bad(1, s);
        GNNA_CUDA(cudaMemsetAsync(owner.get(), 0xff, (size_t)n * 4, s));
        GNNA_CUDA(cudaMemsetAsync(bad.get(), 0, 4, s));
        k7_perm_claim<<<gnna::grid_for(n, 256), 256, 0, s>>>(d_vec, n, owner.get(), bad.get());
        gnna::launched(ctx, "k7_perm_claim");
        if (read_flag(ctx, bad)) gnna::raise(GNNA_ERR_DOMAIN, "mapping is not a permutation of its index range");
        if (d_old_to_new != d_vec)
            GNNA_CUDA(cudaMemcpyAsync(d_old_to_new, d_vec, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
        k7_copy_u32<<<gnna::grid_for(n, 256), 256, 0, s>>>(owner.get(), n, d_new_to_old);
        gnna::launched(ctx, "k7_copy_u32");
        GNNA_CUDA(cudaStreamSynchronize(s));
    });
}

gnna_status gnna_apply_mapping_csr(gnna_ctx* ctx, const uint64_t* d_row_ptr, const uint32_t* d_col, uint32_t n,
                                   const uint32_t* d_old_to_new, const uint32_t* d_new_to_old, uint64_t* d_out_row_ptr,
                                   uint32_t* d_out_col) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        cudaStream_t s = ctx->stream;
        if (n) {
            DevBuf<unsigned> bad(1, s);
            GNNA_CUDA(cudaMemsetAsync(bad.get(), 0, 4, s));
            k7_check_mapping<<<gnna::grid_for(n, 256), 256, 0, s>>>(d_old_to_new, d_new_to_old, n, bad.get());
            gnna::launched(ctx, "k7_check_mapping");
            if (read_flag(ctx, bad)) gnna::raise(GNNA_ERR_DOMAIN, "apply_mapping: mapping is not a permutation");
        }
        uint64_t m = 0;
        gnna::to_host(ctx, &m, d_row_ptr + n, 1);
        DevBuf<uint64_t> keys(m ? m : 1, s);
        if (m) {
            k7_relabel_keys<<<gnna::grid_for((uint64_t)n * 32, 256), 256, 0, s>>>(d_row_ptr, d_col, n, d_old_to_new,
                                                                                  keys.get());
            gnna::launched(ctx, "k7_relabel_keys");
        }
        gnna::csr_from_keys(ctx, keys.get(), m, n, d_out_row_ptr, d_out_col, false);
        GNNA_CUDA(cudaStreamSynchronize(s));
    });
}

gnna_status gnna_apply_mapping_edges(gnna_ctx* ctx, const uint32_t* d_edges, uint64_t e, uint32_t n,
                                     const uint32_t* d_old_to_new, uint32_t* d_out_edges) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (!e) return;
        cudaStream_t s = ctx->stream;
        DevBuf<unsigned> bad(1, s);
        GNNA_CUDA(cudaMemsetAsync(bad.get(), 0, 4, s));
        k7_relabel_edges<<<gnna::grid_for(e, 256), 256, 0, s>>>(d_edges, e, n, d_old_to_new, d_out_edges, bad.get());
        gnna::launched(ctx, "k7_relabel_edges");
        if (read_flag(ctx, bad)) gnna::raise(GNNA_ERR_DOMAIN, "apply_mapping: edge endpoint out of range");
    });
}

gnna_status gnna_hub_remap(gnna_ctx* ctx, const uint64_t* d_row_ptr, const uint32_t* d_col, uint32_t n, uint32_t k,
                           uint32_t* d_hubs, uint32_t* d_col_out, uint64_t* hub_edges) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (k > n) gnna::raise(GNNA_ERR_DOMAIN, "hub_remap: more hubs than nodes");
        if ((uint64_t)n + k > 0xffffffffull) gnna::raise(GNNA_ERR_DOMAIN, "hub_remap: n + k must fit in 32 bits");
        cudaStream_t s = ctx->stream;
        uint64_t nnz = 0;
        if (n) gnna::to_host(ctx, &nnz, d_row_ptr + n, 1);
        DevBuf<uint32_t> slot(n ? n : 1, s);
        DevBuf<unsigned long long> hits(1, s);
        GNNA_CUDA(cudaMemsetAsync(slot.get(), 0xff, (size_t)(n ? n : 1) * 4, s));
        GNNA_CUDA(cudaMemsetAsync(hits.get(), 0, 8, s));
        if (k) {  // the k highest-degree nodes, ties by id (the gnna_degree_order keys)
            DevBuf<uint64_t> keys(n, s);
            k7_degree_keys<<<gnna::grid_for(n, 256), 256, 0, s>>>(d_row_ptr, n, keys.get());
            gnna::launched(ctx, "k7_degree_keys");
            gnna::sort_keys_u64(ctx, keys.get(), n, 64);
            k7_hub_slots<<<gnna::grid_for(k, 256), 256, 0, s>>>(keys.get(), k, d_hubs, slot.get());
            gnna::launched(ctx, "k7_hub_slots");
        }
        if (nnz) {
            k7_hub_remap<<<gnna::grid_for(nnz, 256), 256, 0, s>>>(d_col, nnz, slot.get(), n, d_col_out, hits.get());
            gnna::launched(ctx, "k7_hub_remap");
        }
        unsigned long long h = 0;
        gnna::to_host(ctx, &h, hits.get(), 1);
        if (hub_edges) *hub_edges = h;
    });
}

gnna_status gnna_gather_rows(gnna_ctx* ctx, int dtype, const void* d_x, uint32_t dim, const uint32_t* d_rows,
                             uint64_t count, void* d_out) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (dtype != GNNA_F32 && dtype != GNNA_F64) gnna::raise(GNNA_ERR_DOMAIN, "unknown dtype");
        const uint64_t total = count * dim;
        if (!total) return;
        if (dtype == GNNA_F32)
            k7_gather_rows<float><<<gnna::grid_for(total, 256), 256, 0, ctx->stream>>>(
                static_cast<const float*>(d_x), dim, d_rows, count, static_cast<float*>(d_out));
        else
            k7_gather_rows<double><<<gnna::grid_for(total, 256), 256, 0, ctx->stream>>>(
                static_cast<const double*>(d_x), dim, d_rows, count, static_cast<double*>(d_out));
        gnna::launched(ctx, "k7_gather_rows");
    });
}

gnna_status gnna_b200_plan_params(gnna_ctx* ctx, const uint64_t* d_row_ptr, uint32_t n, uint32_t dim, int dtype,
                                  double hbm_gbs, gnna_params* out, double* est_us, uint64_t* l2_window_bytes) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (!out) gnna::raise(GNNA_ERR_DOMAIN, "b200_plan_params: null output");
        if (dtype != GNNA_F32 && dtype != GNNA_F64) gnna::raise(GNNA_ERR_DOMAIN, "unknown dtype");
        if (dim == 0) gnna::raise(GNNA_ERR_DOMAIN, "dim must be positive");
        cudaStream_t s = ctx->stream;
        gnna_decider::B200Inputs g{};
        g.num_nodes = n;
        g.dim = dim;
        g.elem = dtype == GNNA_F32 ? 4 : 8;
        g.num_sms = (uint32_t)ctx->num_sms;
        g.l2_bytes = ctx->l2_bytes > 0 ? (uint64_t)ctx->l2_bytes : 0;
        g.hbm_gbs = hbm_gbs;
        const uint64_t row = (uint64_t)dim * g.elem, l2 = g.l2_bytes ? g.l2_bytes : 126500000ull;
        g.window_bytes = 48ull << 20;
        if (n) {
            gnna::to_host(ctx, &g.num_edges, d_row_ptr + n, 1);
            DevBuf<uint64_t> keys(n, s);
            k7_degree_keys<<<gnna::grid_for(n, 256), 256, 0, s>>>(d_row_ptr, n, keys.get());
            gnna::launched(ctx, "k7_degree_keys");
            gnna::sort_keys_u64(ctx, keys.get(), n, 64);
            uint64_t k0 = 0;
            gnna::to_host(ctx, &k0, keys.get(), 1);
            g.max_degree = (uint32_t)~(uint32_t)(k0 >> 32);
            // gather shares (symmetric CSR: in-degree = degree) of the rows that fit in L2/2 and in the window
            const uint64_t kl2 = std::min<uint64_t>(n, l2 / 2 / row), kw = std::min<uint64_t>(n, g.window_bytes / row);
            DevBuf<unsigned long long> sums(2, s);
            GNNA_CUDA(cudaMemsetAsync(sums.get(), 0, 16, s));
            if (kl2) k7_topk_degree_sum<<<gnna::grid_for(kl2, 256), 256, 0, s>>>(keys.get(), kl2, sums.get());
            if (kw) k7_topk_degree_sum<<<gnna::grid_for(kw, 256), 256, 0, s>>>(keys.get(), kw, sums.get() + 1);
            gnna::launched(ctx, "k7_topk_degree_sum");
            unsigned long long h[2] = {0, 0};
            gnna::to_host(ctx, h, sums.get(), 2);
            const double nnz = g.num_edges ? (double)g.num_edges : 1.0;
            g.l2_hit_share = h[0] / nnz;
            g.window_share = h[1] / nnz;
            g.window_rows_frac = (double)kw / n;
        }
        try {
            *out = gnna_decider::b200_params(g, est_us, l2_window_bytes);
        } catch (const gnna_decider::Domain& d) {
            gnna::raise(GNNA_ERR_DOMAIN, d.msg);
        }
    });
}

}  // extern "C"
