// K6: the node update X·W (engine.cpp:315-331 matmul) and the transposed
// products of the backward pass, for sm_100a.
//
// Shapes on this path are skinny: m = nodes (10^5..10^7), k and n = feature
// widths (<= a few hundred).  At C3 (410k x 96 · 96 x 16) the product moves
// 158 MB for 1.3 GFLOP (8 flop/B): it is HBM-bound, so the kernel is a
// streaming SIMT kernel (coalesced A tiles staged in shared memory, W resident
// in shared memory, one output row per thread) rather than a tensor-core
// tile.  tcgen05 kind::tf32 would also break the 1e-5 fp32 parity bar
// (SURVEY §7 hard part 5) for no speed gain at 8 flop/B.
//
// GEMM_EXACT (fp64 API): per output element the reference's order — k
// ascending, a == 0 skipped, a separately rounded product added to the
// running sum starting from 0.0 — so results are bitwise equal to matmul.
//
// gemm_tn (dW = A^T B, a reduction over all rows) is split over row chunks
// with per-chunk partials summed in chunk order: deterministic.
#include <algorithm>

#include "gnna_common.cuh"

namespace {

using gnna::DevBuf;

__device__ __forceinline__ double fmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double fadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }

constexpr int ROWS = 128;  // rows per CTA (one per thread)
constexpr int KC = 32;     // k chunk staged per pass
constexpr int NJ = 32;     // output columns per pass (registers)

struct GemmArgs {
    const void* a;
    const void* w;
    const void* bias;
    const double* row_scale;
    void* out;
    uint32_t m, k, n;
    int epilogue;  // 0 none, 1 bias + relu, 2 row scale
};

// out[i, j0:j0+NJ] = sum_k a[i,k] w[k,j]   (+ epilogue)
template <class T, bool EXACT>
__global__ void __launch_bounds__(ROWS) k6_gemm(GemmArgs g) {
    __shared__ T sa[ROWS][KC + 1];
    __shared__ T sw[KC][NJ];
    const T* __restrict__ a = static_cast<const T*>(g.a);
    const T* __restrict__ w = static_cast<const T*>(g.w);
    const uint64_t row0 = (uint64_t)blockIdx.x * ROWS;
    const uint32_t j0 = blockIdx.y * NJ;
    const uint32_t nj = g.n - j0 < (uint32_t)NJ ? g.n - j0 : (uint32_t)NJ;
    const uint32_t t = threadIdx.x;
    T acc[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[j] = T(0);
    for (uint32_t k0 = 0; k0 < g.k; k0 += KC) {
        const uint32_t kc = g.k - k0 < (uint32_t)KC ? g.k - k0 : (uint32_t)KC;
        // stage A[row0:row0+ROWS, k0:k0+kc] (coalesced along k)
        for (uint32_t e = t; e < ROWS * KC; e += ROWS) {
            const uint32_t r = e / KC, c = e % KC;
            const uint64_t gr = row0 + r;
            sa[r][c] = (gr < g.m && c < kc) ? a[gr * g.k + k0 + c] : T(0);
        }
        for (uint32_t e = t; e < KC * NJ; e += ROWS) {
            const uint32_t r = e / NJ, c = e % NJ;
            sw[r][c] = (r < kc && c < nj) ? w[(uint64_t)(k0 + r) * g.n + j0 + c] : T(0);
        }
        __syncthreads();
        for (uint32_t kk = 0; kk < kc; ++kk) {
            const T av = sa[t][kk];
            if (EXACT) {
                if (av == T(0)) continue;  // engine.cpp:325 `if (aik == 0.0) continue;`
#pragma unroll
                for (int j = 0; j < NJ; ++j) acc[j] = fadd(acc[j], fmul(av, sw[kk][j]));
            } else {
#pragma unroll
                for (int j = 0; j < NJ; ++j) acc[j] += av * sw[kk][j];
            }
        }
        __syncthreads();
    }
    const uint64_t r = row0 + t;
    if (r >= g.m) return;
    T* o = static_cast<T*>(g.out) + r * g.n + j0;
    if (g.epilogue == 1) {
        const T* b = static_cast<const T*>(g.bias) + j0;
#pragma unroll
        for (int j = 0; j < NJ; ++j)
            if (j < (int)nj) {
                const T v = EXACT ? fadd(acc[j], b[j]) : acc[j] + b[j];
                o[j] = v > T(0) ? v : T(0);  // std::max(0.0, h + b)
            }
    } else if (g.epilogue == 2) {
        const T s = T(g.row_scale[r]);
#pragma unroll
        for (int j = 0; j < NJ; ++j)
            if (j < (int)nj) o[j] = EXACT ? fmul(s, acc[j]) : s * acc[j];
    } else {
#pragma unroll
        for (int j = 0; j < NJ; ++j)
            if (j < (int)nj) o[j] = acc[j];
    }
}

// Partial C = A[rows]^T B[rows] for one chunk of rows: A m x p, B m x q.
// grid.x = row chunks, grid.y = output tiles of TN_OUT elements.
constexpr int TN_THREADS = 256;
constexpr int TN_PER = 8;
constexpr int TN_OUT = TN_THREADS * TN_PER;
constexpr int TN_ROWS = 16;

template <class T>
__global__ void __launch_bounds__(TN_THREADS) k6_gemm_tn_partial(const T* __restrict__ a, const T* __restrict__ b,
                                                                 uint32_t m, uint32_t p, uint32_t q,
                                                                 uint32_t rows_per_chunk, T* __restrict__ part) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sa = reinterpret_cast<T*>(smem_raw);      // [TN_ROWS][p]
    T* sb = sa + (size_t)TN_ROWS * p;            // [TN_ROWS][q]
    const uint64_t r_begin = (uint64_t)blockIdx.x * rows_per_chunk;
    const uint64_t r_end = r_begin + rows_per_chunk < m ? r_begin + rows_per_chunk : m;
    const uint32_t o0 = blockIdx.y * TN_OUT;
    const uint32_t total = p * q;
    T acc[TN_PER];
    uint32_t oi[TN_PER], oj[TN_PER];
#pragma unroll
    for (int s = 0; s < TN_PER; ++s) {
        acc[s] = T(0);
        const uint32_t o = o0 + threadIdx.x + s * TN_THREADS;
        oi[s] = o < total ? o / q : 0;
        oj[s] = o < total ? o % q : 0;
    }
    for (uint64_t r0 = r_begin; r0 < r_end; r0 += TN_ROWS) {
        const uint32_t nr = (uint32_t)(r_end - r0 < (uint64_t)TN_ROWS ? r_end - r0 : (uint64_t)TN_ROWS);
        for (uint32_t e = threadIdx.x; e < TN_ROWS * p; e += TN_THREADS) {
            const uint32_t r = e / p;
            sa[e] = r < nr ? a[(r0 + r) * p + e % p] : T(0);
        }
        for (uint32_t e = threadIdx.x; e < TN_ROWS * q; e += TN_THREADS) {
            const uint32_t r = e / q;
            sb[e] = r < nr ? b[(r0 + r) * q + e % q] : T(0);
        }
        __syncthreads();
        for (uint32_t r = 0; r < nr; ++r) {
#pragma unroll
            for (int s = 0; s < TN_PER; ++s) acc[s] += sa[r * p + oi[s]] * sb[r * q + oj[s]];
        }
        __syncthreads();
    }
#pragma unroll
    for (int s = 0; s < TN_PER; ++s) {
        const uint32_t o = o0 + threadIdx.x + s * TN_THREADS;
        if (o < total) part[(size_t)blockIdx.x * total + o] = acc[s];
    }
}

// out[o] = sum over chunks (in chunk order) of part[c][o]  (+= when accumulate)
template <class T>
__global__ void k6_reduce_chunks(const T* __restrict__ part, uint32_t chunks, uint32_t total, T* __restrict__ out) {
    for (uint32_t o = blockIdx.x * blockDim.x + threadIdx.x; o < total; o += gridDim.x * blockDim.x) {
        T s = T(0);
        for (uint32_t c = 0; c < chunks; ++c) s += part[(size_t)c * total + o];
        out[o] = s;
    }
}

template <class T>
__global__ void k6_transpose(const T* __restrict__ w, uint32_t rows, uint32_t cols, T* __restrict__ wt) {
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols; e += gridDim.x * blockDim.x) {
        const uint32_t r = e / cols, c = e % cols;
        wt[(size_t)c * rows + r] = w[e];
    }
}

// Column sums of B (m x q), chunked and reduced in order: db = sum_rows dU.
template <class T>
__global__ void k6_colsum_partial(const T* __restrict__ b, uint32_t m, uint32_t q, uint32_t rows_per_chunk,
                                  T* __restrict__ part) {
    const uint64_t r_begin = (uint64_t)blockIdx.x * rows_per_chunk;
    const uint64_t r_end = r_begin + rows_per_chunk < m ? r_begin + rows_per_chunk : m;
    for (uint32_t j = threadIdx.x; j < q; j += blockDim.x) {
        T s = T(0);
        for (uint64_t r = r_begin; r < r_end; ++r) s += b[r * q + j];
        part[(size_t)blockIdx.x * q + j] = s;
    }
}

template <class T>
void launch_gemm(gnna_ctx* ctx, const GemmArgs& g, bool exact) {
    if (g.m == 0 || g.n == 0) return;
    dim3 grid((g.m + ROWS - 1) / ROWS, (g.n + NJ - 1) / NJ);
    if (exact)
        k6_gemm<T, true><<<grid, ROWS, 0, ctx->stream>>>(g);
    else
        k6_gemm<T, false><<<grid, ROWS, 0, ctx->stream>>>(g);
    gnna::launched(ctx, "k6_gemm");
}

template <class T>
void launch_gemm_tn(gnna_ctx* ctx, const T* a, const T* b, uint32_t m, uint32_t p, uint32_t q, T* out) {
    const uint32_t total = p * q;
    if (total == 0) return;
    if (m == 0) {
        GNNA_CUDA(cudaMemsetAsync(out, 0, (size_t)total * sizeof(T), ctx->stream));
        return;
    }
    const uint32_t tiles = (total + TN_OUT - 1) / TN_OUT;
    uint32_t chunks = std::max<uint32_t>(1, std::min<uint32_t>(4 * ctx->num_sms / tiles + 1, (m + 255) / 256));
    const uint32_t rpc = (m + chunks - 1) / chunks;
    chunks = (m + rpc - 1) / rpc;
    DevBuf<T> part((size_t)chunks * total, ctx->stream);
    const size_t smem = (size_t)TN_ROWS * (p + q) * sizeof(T);
    if (smem > 200 * 1024) gnna::raise(GNNA_ERR_DOMAIN, "gemm_tn: feature widths too large");
    if (smem > 48 * 1024)
        GNNA_CUDA(cudaFuncSetAttribute(k6_gemm_tn_partial<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k6_gemm_tn_partial<T><<<dim3(chunks, tiles), TN_THREADS, smem, ctx->stream>>>(a, b, m, p, q, rpc, part.get());
    gnna::launched(ctx, "k6_gemm_tn_partial");
    k6_reduce_chunks<T><<<gnna::grid_for(total, 256), 256, 0, ctx->stream>>>(part.get(), chunks, total, out);
    gnna::launched(ctx, "k6_reduce_chunks");
}

}  // namespace

namespace gnna {

// out = a (m x k) . w (k x n)  [+ epilogue]; exact => reference order (f64).
void gemm(gnna_ctx* ctx, int dtype, const void* a, uint32_t m, uint32_t k, const void* w, uint32_t n,
          const void* bias, int epilogue, const double* row_scale, void* out) {
    GemmArgs g{a, w, bias, row_scale, out, m, k, n, epilogue};
    if (epilogue == 1 && !bias) raise(GNNA_ERR_DOMAIN, "gemm: bias epilogue without a bias");
    if (epilogue == 2 && !row_scale) raise(GNNA_ERR_DOMAIN, "gemm: row-scale epilogue without scales");
    if (dtype == GNNA_F32)
        launch_gemm<float>(ctx, g, false);
    else if (dtype == GNNA_F64)
        launch_gemm<double>(ctx, g, true);
    else
        raise(GNNA_ERR_DOMAIN, "unknown dtype");
}

// out (p x q) = a^T b with a: m x p, b: m x q (deterministic chunked reduction).
void gemm_tn(gnna_ctx* ctx, int dtype, const void* a, const void* b, uint32_t m, uint32_t p, uint32_t q, void* out) {
    if (dtype == GNNA_F32)
        launch_gemm_tn<float>(ctx, static_cast<const float*>(a), static_cast<const float*>(b), m, p, q,
                              static_cast<float*>(out));
    else
        launch_gemm_tn<double>(ctx, static_cast<const double*>(a), static_cast<const double*>(b), m, p, q,
                               static_cast<double*>(out));
}

// wt (cols x rows) = w^T
void transpose(gnna_ctx* ctx, int dtype, const void* w, uint32_t rows, uint32_t cols, void* wt) {
    if ((uint64_t)rows * cols == 0) return;
    if (dtype == GNNA_F32)
        k6_transpose<float><<<grid_for((uint64_t)rows * cols, 256), 256, 0, ctx->stream>>>(
            static_cast<const float*>(w), rows, cols, static_cast<float*>(wt));
    else
        k6_transpose<double><<<grid_for((uint64_t)rows * cols, 256), 256, 0, ctx->stream>>>(
            static_cast<const double*>(w), rows, cols, static_cast<double*>(wt));
    launched(ctx, "k6_transpose");
}

// out (q) = column sums of b (m x q), deterministic.
void colsum(gnna_ctx* ctx, int dtype, const void* b, uint32_t m, uint32_t q, void* out) {
    if (q == 0) return;
    const size_t es = dtype == GNNA_F32 ? 4 : 8;
    if (m == 0) {
        GNNA_CUDA(cudaMemsetAsync(out, 0, q * es, ctx->stream));
        return;
    }
    uint32_t chunks = std::min<uint32_t>(4 * ctx->num_sms, (m + 63) / 64);
    const uint32_t rpc = (m + chunks - 1) / chunks;
    chunks = (m + rpc - 1) / rpc;
    DevBuf<uint8_t> part((size_t)chunks * q * es, ctx->stream);
    const unsigned th = std::min<uint32_t>(256, ((q + 31) / 32) * 32);
    if (dtype == GNNA_F32) {
        k6_colsum_partial<float><<<chunks, th, 0, ctx->stream>>>(static_cast<const float*>(b), m, q, rpc,
                                                                 reinterpret_cast<float*>(part.get()));
        launched(ctx, "k6_colsum_partial");
        k6_reduce_chunks<float><<<grid_for(q, 256), 256, 0, ctx->stream>>>(reinterpret_cast<float*>(part.get()),
                                                                           chunks, q, static_cast<float*>(out));
    } else {
        k6_colsum_partial<double><<<chunks, th, 0, ctx->stream>>>(static_cast<const double*>(b), m, q, rpc,
                                                                  reinterpret_cast<double*>(part.get()));
        launched(ctx, "k6_colsum_partial");
        k6_reduce_chunks<double><<<grid_for(q, 256), 256, 0, ctx->stream>>>(
            reinterpret_cast<double*>(part.get()), chunks, q, static_cast<double*>(out));
    }
    launched(ctx, "k6_reduce_chunks");
}

}  // namespace gnna

extern "C" gnna_status gnna_gemm(gnna_ctx* ctx, int dtype, const void* d_a, uint32_t m, uint32_t k, const void* d_w,
                                 uint32_t n_out, const void* d_bias, int epilogue, const double* d_row_scale,
                                 void* d_out) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        gnna::gemm(ctx, dtype, d_a, m, k, d_w, n_out, d_bias, epilogue, d_row_scale, d_out);
    });
}

extern "C" gnna_status gnna_gemm_tn(gnna_ctx* ctx, int dtype, const void* d_a, const void* d_b, uint32_t m, uint32_t p,
                                    uint32_t q, void* d_out) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (dtype != GNNA_F32 && dtype != GNNA_F64) gnna::raise(GNNA_ERR_DOMAIN, "unknown dtype");
        gnna::gemm_tn(ctx, dtype, d_a, d_b, m, p, q, d_out);
    });
}
