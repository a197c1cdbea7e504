// Graph utilities on the GPU: to_csr (graph.cpp:76-95), CSR transpose,
// aes (graph.cpp:122-128), degree_stats (graph.cpp:106-120) and
// ModelInputs::from_graph (decider.cpp:26-37).
//
// to_csr: every (src,dst) edge (plus (dst,src) when symmetrising) becomes one
// u64 key row<<32|col; an LSD radix sort over the used bits orders rows and
// columns at once, a flag+scan drops duplicates (the reference's sort+unique
// per row) and a per-row count + scan gives row_ptr.  Self loops are kept,
// exactly like the reference.  Integer outputs are bit-exact.
#include <cub/device/device_select.cuh>

#include <cmath>
#include <vector>

#include "gnna_common.cuh"

namespace {

using gnna::DevBuf;

int bits_for(uint64_t v) {
    int b = 0;
    while (b < 64 && (v >> b)) ++b;
    return b < 1 ? 1 : b;
}

__global__ void k_edge_keys(const uint32_t* __restrict__ edges, uint64_t e, int sym, uint32_t n,
                            uint64_t* __restrict__ keys, unsigned* __restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < e; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint2 uv = reinterpret_cast<const uint2*>(edges)[i];
        if (uv.x >= n || uv.y >= n) atomicExch(bad, 1u);
        keys[sym ? 2 * i : i] = ((uint64_t)uv.x << 32) | uv.y;
        if (sym) keys[2 * i + 1] = ((uint64_t)uv.y << 32) | uv.x;
    }
}

// After the sort: flag the first copy of every key.
__global__ void k_unique_flags(const uint64_t* __restrict__ keys, uint64_t m, uint8_t* __restrict__ keep) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        keep[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// Unique sorted keys -> col (low word); row_ptr[r] = lower_bound(keys, r<<32).
__global__ void k_low_words(const uint64_t* __restrict__ keys, uint64_t m, uint32_t* __restrict__ col) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        col[i] = (uint32_t)keys[i];
}

__global__ void k_row_ptr_bsearch(const uint64_t* __restrict__ keys, uint64_t m, uint32_t n,
                                  uint64_t* __restrict__ row_ptr) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r <= n; r += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t key = r << 32;
        uint64_t lo = 0, hi = m;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (keys[mid] < key) lo = mid + 1; else hi = mid;
        }
        row_ptr[r] = lo;
    }
}

__global__ void k_transpose_keys(const uint64_t* __restrict__ row_ptr, const uint32_t* __restrict__ col, uint32_t n,
                                 uint64_t* __restrict__ keys) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t v = blockIdx.x * (uint64_t)(blockDim.x / 32) + threadIdx.x / 32; v < n; v += warps)
        for (uint64_t p = row_ptr[v] + lane; p < row_ptr[v + 1]; p += 32) keys[p] = ((uint64_t)col[p] << 32) | v;
}

__global__ void k_span_sum(const uint32_t* __restrict__ edges, uint64_t e, unsigned long long* __restrict__ out) {
    unsigned long long s = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < e; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint2 uv = reinterpret_cast<const uint2*>(edges)[i];
        s += uv.x > uv.y ? uv.x - uv.y : uv.y - uv.x;
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

// Per-CTA (max degree, sum of squared deviations) in a fixed reduction order.
__global__ void k_degree_stats(const uint64_t* __restrict__ row_ptr, uint32_t n, double avg,
                               unsigned long long* __restrict__ maxd, double* __restrict__ part) {
    __shared__ double sh[32];
    double sq = 0.0;
    unsigned long long mx = 0;
    const uint64_t per = (n + gridDim.x - 1) / gridDim.x;
    const uint64_t b = blockIdx.x * per, e = b + per < n ? b + per : n;
    for (uint64_t v = b + threadIdx.x; v < e; v += blockDim.x) {
        const uint64_t d = row_ptr[v + 1] - row_ptr[v];
        mx = d > mx ? d : mx;
        const double dc = (double)d - avg;
        sq += dc * dc;
    }
    for (int o = 16; o; o >>= 1) {
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = t > mx ? t : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        sh[threadIdx.x / 32] = sq;
        atomicMax(maxd, mx);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (unsigned w = 0; w < blockDim.x / 32; ++w) s += sh[w];
        part[blockIdx.x] = s;
    }
}

void degree_stats(gnna_ctx* ctx, const uint64_t* row_ptr, uint32_t n, double* avg, uint64_t* maxd, double* sd) {
    if (n == 0) gnna::raise(GNNA_ERR_DOMAIN, "degree_stats: graph has no nodes");
    uint64_t nnz = 0;
    gnna::to_host(ctx, &nnz, row_ptr + n, 1);
    const double a = (double)nnz / (double)n;
    const unsigned grid = std::min<unsigned>(592, (n + 255) / 256);
    DevBuf<unsigned long long> mx(1, ctx->stream);
    DevBuf<double> part(grid, ctx->stream);
    GNNA_CUDA(cudaMemsetAsync(mx.get(), 0, 8, ctx->stream));
    k_degree_stats<<<grid, 256, 0, ctx->stream>>>(row_ptr, n, a, mx.get(), part.get());
    gnna::launched(ctx, "k_degree_stats");
    std::vector<double> h(grid);
    gnna::to_host(ctx, h.data(), part.get(), grid);
    unsigned long long m = 0;
    gnna::to_host(ctx, &m, mx.get(), 1);
    double sq = 0.0;
    for (double v : h) sq += v;
    if (avg) *avg = a;
    if (maxd) *maxd = m;
    if (sd) *sd = std::sqrt(sq / (double)n);
}

}  // namespace

namespace gnna {

// Sorted, de-duplicated CSR from u64 (row<<32|col) keys; keys is clobbered.
// Returns nnz; col must hold `m` entries.
uint64_t csr_from_keys(gnna_ctx* ctx, uint64_t* keys, uint64_t m, uint32_t n, uint64_t* row_ptr, uint32_t* col,
                       bool dedup) {
    cudaStream_t s = ctx->stream;
    const int end_bit = 32 + bits_for(n ? n - 1 : 0);
    sort_keys_u64(ctx, keys, m, end_bit);
    uint64_t nnz = 0;
    if (m && !dedup) {
        nnz = m;
        k_row_ptr_bsearch<<<grid_for((uint64_t)n + 1, 256), 256, 0, s>>>(keys, m, n, row_ptr);
        launched(ctx, "k_row_ptr_bsearch");
        if (col) {
            k_low_words<<<grid_for(m, 256), 256, 0, s>>>(keys, m, col);
            launched(ctx, "k_low_words");
        }
    } else if (m) {
        DevBuf<uint8_t> keep(m, s);
        k_unique_flags<<<grid_for(m, 256), 256, 0, s>>>(keys, m, keep.get());
        launched(ctx, "k_unique_flags");
        DevBuf<uint64_t> uniq(m, s);
        DevBuf<uint64_t> cnt(1, s);
        size_t bytes = 0;
        GNNA_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, keys, keep.get(), uniq.get(), cnt.get(), (int64_t)m, s));
        DevBuf<uint8_t> tmp(bytes, s);
        GNNA_CUDA(cub::DeviceSelect::Flagged(tmp.get(), bytes, keys, keep.get(), uniq.get(), cnt.get(), (int64_t)m, s));
        to_host(ctx, &nnz, cnt.get(), 1);
        k_row_ptr_bsearch<<<grid_for((uint64_t)n + 1, 256), 256, 0, s>>>(uniq.get(), nnz, n, row_ptr);
        launched(ctx, "k_row_ptr_bsearch");
        if (col && nnz) {
            k_low_words<<<grid_for(nnz, 256), 256, 0, s>>>(uniq.get(), nnz, col);
            launched(ctx, "k_low_words");
        }
    } else {
        GNNA_CUDA(cudaMemsetAsync(row_ptr, 0, ((size_t)n + 1) * 8, s));
    }
    return nnz;
}

}  // namespace gnna

extern "C" {

gnna_status gnna_to_csr(gnna_ctx* ctx, uint32_t n, const uint32_t* d_edges, uint64_t e, int symmetrize,
                        uint64_t* d_row_ptr, uint32_t* d_col, uint64_t* nnz) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (!nnz) gnna::raise(GNNA_ERR_DOMAIN, "to_csr: null nnz");
        cudaStream_t s = ctx->stream;
        const uint64_t m = symmetrize ? 2 * e : e;
        DevBuf<uint64_t> keys(m ? m : 1, s);
        DevBuf<unsigned> bad(1, s);
        GNNA_CUDA(cudaMemsetAsync(bad.get(), 0, 4, s));
        if (e) {
            k_edge_keys<<<gnna::grid_for(e, 256), 256, 0, s>>>(d_edges, e, symmetrize, n, keys.get(), bad.get());
            gnna::launched(ctx, "k_edge_keys");
        }
        unsigned b = 0;
        gnna::to_host(ctx, &b, bad.get(), 1);
        if (b) gnna::raise(GNNA_ERR_DOMAIN, "to_csr: edge endpoint out of range");
        DevBuf<uint64_t> rp_tmp;
        uint64_t* rp = d_row_ptr;
        if (!rp) {
            rp_tmp = DevBuf<uint64_t>((uint64_t)n + 1, s);
            rp = rp_tmp.get();
        }
        *nnz = gnna::csr_from_keys(ctx, keys.get(), m, n, rp, d_col, true);
        GNNA_CUDA(cudaStreamSynchronize(s));
    });
}

gnna_status gnna_csr_transpose(gnna_ctx* ctx, const uint64_t* d_row_ptr, const uint32_t* d_col, uint32_t n,
                               uint64_t* d_t_ptr, uint32_t* d_t_col) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        cudaStream_t s = ctx->stream;
        uint64_t m = 0;
        gnna::to_host(ctx, &m, d_row_ptr + n, 1);
        DevBuf<uint64_t> keys(m ? m : 1, s);
        if (m) {
            k_transpose_keys<<<gnna::grid_for((uint64_t)n * 32, 256), 256, 0, s>>>(d_row_ptr, d_col, n, keys.get());
            gnna::launched(ctx, "k_transpose_keys");
        }
        const uint64_t got = gnna::csr_from_keys(ctx, keys.get(), m, n, d_t_ptr, d_t_col, true);
        if (got != m) gnna::raise(GNNA_ERR_DOMAIN, "csr_transpose: input rows have duplicate columns");
        GNNA_CUDA(cudaStreamSynchronize(s));
    });
}

gnna_status gnna_aes(gnna_ctx* ctx, const uint32_t* d_edges, uint64_t e, double* out) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (e == 0) gnna::raise(GNNA_ERR_DOMAIN, "no edges in the input");
        DevBuf<unsigned long long> sum(1, ctx->stream);
        GNNA_CUDA(cudaMemsetAsync(sum.get(), 0, 8, ctx->stream));
        k_span_sum<<<gnna::grid_for(e, 256, 148 * 8), 256, 0, ctx->stream>>>(d_edges, e, sum.get());
        gnna::launched(ctx, "k_span_sum");
        unsigned long long h = 0;
        gnna::to_host(ctx, &h, sum.get(), 1);
        // graph.cpp:124-127 sums the spans in double; the integer sum is the
        // same value while it stays below 2^53.
        if (h >= (1ull << 53)) gnna::raise(GNNA_ERR_DOMAIN, "aes: span sum exceeds 2^53 (not exactly representable)");
        *out = (double)h / (double)e;
    });
}

gnna_status gnna_degree_stats(gnna_ctx* ctx, const uint64_t* d_row_ptr, uint32_t n, double* avg, uint64_t* max_degree,
                              double* stddev) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        degree_stats(ctx, d_row_ptr, n, avg, max_degree, stddev);
    });
}

gnna_status gnna_model_inputs_from_graph(gnna_ctx* ctx, const uint64_t* d_row_ptr, uint32_t n, uint32_t dim,
                                         gnna_model_inputs* out) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (dim == 0) gnna::raise(GNNA_ERR_DOMAIN, "dim must be positive");
        double avg = 0, sd = 0;
        uint64_t mx = 0;
        degree_stats(ctx, d_row_ptr, n, &avg, &mx, &sd);
        gnna_model_inputs in{};
        in.num_nodes = n;
        gnna::to_host(ctx, &in.num_edges, d_row_ptr + n, 1);
        in.dim = dim;
        in.max_tpb = 1024;
        in.avg_degree = avg;
        in.stddev_degree = sd;
        in.smem_per_block = 96 * 1024;
        in.capability = 4096;
        in.alpha = gnna_alpha_from_degrees(avg, sd);
        *out = in;
    });
}

gnna_status gnna_b200_profile(gnna_ctx* ctx, gnna_model_inputs* in) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (!in) gnna::raise(GNNA_ERR_DOMAIN, "null model inputs");
        int tpb = 1024;
        cudaDeviceGetAttribute(&tpb, cudaDevAttrMaxThreadsPerBlock, ctx->device);
        in->max_tpb = (uint32_t)tpb;
        in->smem_per_block = (uint64_t)(ctx->smem_optin ? ctx->smem_optin : 227 * 1024);
    });
}

}  // extern "C"
