// K6: the node update X·W (engine.cpp:315-331 matmul) and the transposed
// products of the backward pass, for sm_100a.
//
// Shapes on this path are skinny: m = nodes (10^5..10^7), k and n = feature
// widths (<= a few hundred).  At C3 (410k x 96 · 96 x 16) the product moves
// 184 MB for 1.3 GFLOP: HBM-bound, but past what fp32 SIMT FMAs sustain at
// HBM speed.  The fp32 product therefore runs on tcgen05 (gemm_tc.cu, 3xTF32
// split so the 1e-5 parity bar holds) for k <= 128; the SIMT kernels below
// (k6_gemm_pipe / k6_gemm_rows / k6_gemm_f32) serve k > 128 and the
// GNNA_GEMM_SIMT=1 A/B switch.
//
// GEMM_EXACT (fp64 API): per output element the reference's order — k
// ascending, a == 0 skipped, a separately rounded product added to the
// running sum starting from 0.0 — so results are bitwise equal to matmul.
//
// gemm_tn (dW = A^T B, a reduction over all rows) is split over row chunks
// with per-chunk partials summed in chunk order: deterministic.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "gnna_common.cuh"

namespace gnna {
bool gemm_tc_f32(gnna_ctx* ctx, const float* a, const float* w, const float* bias, const double* row_scale,
                 float* out, uint32_t m, uint32_t k, uint32_t n, int epilogue);  // gemm_tc.cu
bool gemm_tn_tc_f32(gnna_ctx* ctx, const float* a, const float* b, uint32_t m, uint32_t p, uint32_t q,
                    float* out);  // gemm_tc.cu
}

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

// ------------------------------------------------------ fp32 fast kernels
// X·W for skinny W (n <= 32): one output row per thread, A staged through
// shared memory in coalesced 32-column chunks (row stride 33: conflict-free
// column reads), W chunk in shared memory read as float4 broadcasts, NJ
// accumulators in registers (NJ = n rounded up to 4, 8, 16 or 32).  Per k:
// 1 + NJ/4 shared loads for NJ FMAs; the kernel streams A at HBM speed.
template <int NJ>
__global__ void __launch_bounds__(ROWS) k6_gemm_f32(GemmArgs g) {
    __shared__ float sa[ROWS][KC + 1];
    __shared__ __align__(16) float sw[KC][NJ];
    const float* __restrict__ a = static_cast<const float*>(g.a);
    const float* __restrict__ w = static_cast<const float*>(g.w);
    const uint64_t row0 = (uint64_t)blockIdx.x * ROWS;
    const uint32_t j0 = blockIdx.y * NJ;
    const uint32_t nj = g.n - j0 < (uint32_t)NJ ? g.n - j0 : (uint32_t)NJ;
    const uint32_t t = threadIdx.x;
    float acc[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[j] = 0.f;
    const bool vec4 = (g.k % 4 == 0) && ((uintptr_t)a % 16 == 0);
    for (uint32_t k0 = 0; k0 < g.k; k0 += KC) {
        const uint32_t kc = g.k - k0 < (uint32_t)KC ? g.k - k0 : (uint32_t)KC;
        if (vec4) {
            // 8 independent 16-byte loads per thread in flight (ROWS x KC / 4 / ROWS)
            float4 v[ROWS * KC / 4 / ROWS];
#pragma unroll
            for (int i = 0; i < ROWS * KC / 4 / ROWS; ++i) {
                const uint32_t e = t + i * ROWS;
                const uint32_t r = e / (KC / 4), c4 = e % (KC / 4);
                const uint64_t gr = row0 + r;
                v[i] = (gr < g.m && c4 * 4 < kc)
                           ? __ldg(reinterpret_cast<const float4*>(a + gr * g.k + k0) + c4)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int i = 0; i < ROWS * KC / 4 / ROWS; ++i) {
                const uint32_t e = t + i * ROWS;
                const uint32_t r = e / (KC / 4), c = (e % (KC / 4)) * 4;
                sa[r][c] = v[i].x;
                sa[r][c + 1] = v[i].y;
                sa[r][c + 2] = v[i].z;
                sa[r][c + 3] = v[i].w;
            }
        } else {
#pragma unroll 4
            for (uint32_t e = t; e < ROWS * KC; e += ROWS) {
                const uint32_t r = e / KC, c = e % KC;
                const uint64_t gr = row0 + r;
                sa[r][c] = (gr < g.m && c < kc) ? __ldg(a + gr * g.k + k0 + c) : 0.f;
            }
        }
        for (uint32_t e = t; e < KC * NJ; e += ROWS) {
            const uint32_t r = e / NJ, c = e % NJ;
            sw[r][c] = (r < kc && c < nj) ? __ldg(w + (uint64_t)(k0 + r) * g.n + j0 + c) : 0.f;
        }
        __syncthreads();
#pragma unroll 8
        for (uint32_t kk = 0; kk < (uint32_t)KC; ++kk) {
            const float av = sa[t][kk];
#pragma unroll
            for (int j = 0; j < NJ; j += 4) {
                const float4 w4 = *reinterpret_cast<const float4*>(&sw[kk][j]);
                acc[j] = fmaf(av, w4.x, acc[j]);
                acc[j + 1] = fmaf(av, w4.y, acc[j + 1]);
                acc[j + 2] = fmaf(av, w4.z, acc[j + 2]);
                acc[j + 3] = fmaf(av, w4.w, acc[j + 3]);
            }
        }
        __syncthreads();
    }
    const uint64_t r = row0 + t;
    if (r >= g.m) return;
    float* o = static_cast<float*>(g.out) + r * g.n + j0;
    const float* b = g.epilogue == 1 ? static_cast<const float*>(g.bias) + j0 : nullptr;
    const float s = g.epilogue == 2 ? (float)g.row_scale[r] : 1.f;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        if (j >= (int)nj) break;
        float v = acc[j];
        if (g.epilogue == 1) {
            v += b[j];
            v = v > 0.f ? v : 0.f;
        } else if (g.epilogue == 2) {
            v *= s;
        }
        o[j] = v;
    }
}

// X·W for narrow widths whose rows are not 16-byte multiples (k <= 32,
// k % 4 != 0, n <= 32: the C3 output layer's 22 columns in dZ = dY·W2^T), so
// TMA cannot tile A.  A CTA's 128 rows of A are ONE contiguous run of 128·k floats,
// 16-byte aligned whatever k is, so they are streamed with flat float4 loads
// and scattered into shared memory at an odd row pitch (conflict-free
// row-per-thread reads).  The 128·n outputs go back the same way: staged at
// an odd pitch, stored as one flat float4 run.  FFMA in k order.
constexpr int FL_ROWS = 128, FL_K = 32, FL_LD = FL_ROWS * FL_K / 4 / FL_ROWS;
// Persistent: a CTA walks tiles blockIdx.x, +gridDim.x, ... and issues the
// next tile's A loads before computing the current one (latency overlap).
template <int NJ>
__global__ void __launch_bounds__(FL_ROWS) k6_gemm_flat(GemmArgs g) {
    __shared__ float sa[FL_ROWS * (FL_K + 1)];
    __shared__ float so[FL_ROWS * (FL_K + 1)];
    __shared__ __align__(16) float sw[FL_K * NJ];
    const uint32_t k = g.k, n = g.n, kp = k | 1u, np = n | 1u, t = threadIdx.x;
    // f / k for f < 128·32 without integer division: (f + 0.5)·(1/k) is at
    // least 0.5/k >= 1/64 from the next integer, far above the float error.
    const float rk = 1.f / (float)(k ? k : 1), rn = 1.f / (float)n;
    auto spos = [](uint32_t f, uint32_t w, float rw, uint32_t pitch) {
        const uint32_t r = (uint32_t)(((float)f + 0.5f) * rw);
        return r * pitch + (f - r * w);
    };
    const uint64_t tiles = (g.m + FL_ROWS - 1) / FL_ROWS;
    auto tile_rows = [&](uint64_t tile) {
        const uint64_t r0 = tile * FL_ROWS;
        return g.m - r0 < (uint64_t)FL_ROWS ? (uint32_t)(g.m - r0) : (uint32_t)FL_ROWS;
    };
    float4 v[FL_LD];
    auto load = [&](uint64_t tile) {
        const float4* a4 = reinterpret_cast<const float4*>(static_cast<const float*>(g.a) + tile * FL_ROWS * k);
        const uint32_t nv = tile_rows(tile) * k / 4;
#pragma unroll
        for (int i = 0; i < FL_LD; ++i) {
            const uint32_t e = t + i * FL_ROWS;
            if (e < nv) v[i] = __ldg(a4 + e);
        }
    };
    for (uint32_t e = t; e < FL_K * NJ; e += FL_ROWS) {
        const uint32_t r = e / NJ, c = e % NJ;
        sw[e] = (r < k && c < n) ? __ldg(static_cast<const float*>(g.w) + (uint64_t)r * n + c) : 0.f;
    }
    uint64_t tile = blockIdx.x;
    if (tile < tiles) load(tile);
    for (; tile < tiles; tile += gridDim.x) {
        const uint64_t row0 = tile * FL_ROWS;
        const uint32_t rows = tile_rows(tile);
        const float* __restrict__ a = static_cast<const float*>(g.a) + row0 * k;
        const uint32_t cnt = rows * k, nv = cnt / 4;
#pragma unroll
        for (int i = 0; i < FL_LD; ++i) {
            const uint32_t e = t + i * FL_ROWS;
            if (e < nv) {
                const float x[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) sa[spos(e * 4 + q, k, rk, kp)] = x[q];
            }
        }
        for (uint32_t f = nv * 4 + t; f < cnt; f += FL_ROWS) sa[spos(f, k, rk, kp)] = a[f];
        __syncthreads();
        if (tile + gridDim.x < tiles) load(tile + gridDim.x);
        if (t < rows) {
            float2 acc[NJ / 2];  // column pairs on packed FFMA2 (per-lane fmaf: the same roundings)
#pragma unroll
            for (int j = 0; j < NJ / 2; ++j) acc[j] = make_float2(0.f, 0.f);
            const float* ar = sa + t * kp;
#pragma unroll 4
            for (uint32_t kk = 0; kk < k; ++kk) {
                const float2 av = make_float2(ar[kk], ar[kk]);
#pragma unroll
                for (int j = 0; j < NJ; j += 4) {
                    const float4 w4 = *reinterpret_cast<const float4*>(&sw[kk * NJ + j]);
                    acc[j / 2] = __ffma2_rn(av, make_float2(w4.x, w4.y), acc[j / 2]);
                    acc[j / 2 + 1] = __ffma2_rn(av, make_float2(w4.z, w4.w), acc[j / 2 + 1]);
                }
            }
            const float s = g.epilogue == 2 ? (float)g.row_scale[row0 + t] : 1.f;
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                if (j >= (int)n) break;
                float val = j % 2 ? acc[j / 2].y : acc[j / 2].x;
                if (g.epilogue == 1) {
                    val += static_cast<const float*>(g.bias)[j];
                    val = val > 0.f ? val : 0.f;
                } else if (g.epilogue == 2) {
                    val *= s;
                }
                so[t * np + j] = val;
            }
        }
        __syncthreads();
        float* __restrict__ o = static_cast<float*>(g.out) + row0 * n;
        const uint32_t ocnt = rows * n, onv = ocnt / 4;
        for (uint32_t e = t; e < onv; e += FL_ROWS) {
            float x[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) x[q] = so[spos(e * 4 + q, n, rn, np)];
            reinterpret_cast<float4*>(o)[e] = make_float4(x[0], x[1], x[2], x[3]);
        }
        for (uint32_t f = onv * 4 + t; f < ocnt; f += FL_ROWS) o[f] = so[spos(f, n, rn, np)];
        // sa/so are rewritten by the next tile: no thread may still be reading them
        __syncthreads();
    }
}

// X·W, row per thread with DIRECT 16-byte loads of the thread's own A row
// (no A staging, no barriers in the k loop): a warp instruction reads 16 B of
// 32 rows, the next instruction the following 16 B (L1 hits), so DRAM sees
// each A byte once while every thread keeps KCH/4 loads in flight, and the
// next k chunk is prefetched while the current one is consumed.  W lives in
// shared memory for the whole kernel (read as float4 broadcasts).
// Requires k % 4 == 0, 16-byte aligned A, k*NJ*4 <= 64 KiB.
template <int NJ>
__global__ void __launch_bounds__(128) k6_gemm_rows(GemmArgs g) {
    constexpr int KCH = 16;  // k values per prefetch chunk (4 float4)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* sw = reinterpret_cast<float*>(smem_raw);  // [k][NJ]
    const float* __restrict__ w = static_cast<const float*>(g.w);
    const uint32_t j0 = blockIdx.y * NJ;
    const uint32_t nj = g.n - j0 < (uint32_t)NJ ? g.n - j0 : (uint32_t)NJ;
    for (uint32_t e = threadIdx.x; e < g.k * NJ; e += blockDim.x) {
        const uint32_t r = e / NJ, c = e % NJ;
        sw[e] = c < nj ? __ldg(w + (uint64_t)r * g.n + j0 + c) : 0.f;
    }
    __syncthreads();
    const uint64_t row = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= g.m) return;
    const float4* __restrict__ arow = reinterpret_cast<const float4*>(static_cast<const float*>(g.a) + row * g.k);
    float acc[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[j] = 0.f;
    const uint32_t nch = g.k / KCH, tail = g.k % KCH;
    float4 cur[KCH / 4], nxt[KCH / 4];
    if (nch) {
#pragma unroll
        for (int i = 0; i < KCH / 4; ++i) cur[i] = __ldg(arow + i);
    }
    for (uint32_t ch = 0; ch < nch; ++ch) {
        if (ch + 1 < nch) {
#pragma unroll
            for (int i = 0; i < KCH / 4; ++i) nxt[i] = __ldg(arow + (ch + 1) * (KCH / 4) + i);
        }
        const float* swc = sw + (size_t)ch * KCH * NJ;
#pragma unroll
        for (int i = 0; i < KCH / 4; ++i) {
            const float av[4] = {cur[i].x, cur[i].y, cur[i].z, cur[i].w};
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const float4* w4 = reinterpret_cast<const float4*>(swc + (4 * i + s) * NJ);
#pragma unroll
                for (int j = 0; j < NJ / 4; ++j) {
                    const float4 ww = w4[j];
                    acc[4 * j] = fmaf(av[s], ww.x, acc[4 * j]);
                    acc[4 * j + 1] = fmaf(av[s], ww.y, acc[4 * j + 1]);
                    acc[4 * j + 2] = fmaf(av[s], ww.z, acc[4 * j + 2]);
                    acc[4 * j + 3] = fmaf(av[s], ww.w, acc[4 * j + 3]);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < KCH / 4; ++i) cur[i] = nxt[i];
    }
    for (uint32_t t4 = 0; t4 < tail / 4; ++t4) {
        const float4 v = __ldg(arow + nch * (KCH / 4) + t4);
        const float av[4] = {v.x, v.y, v.z, v.w};
        for (int s = 0; s < 4; ++s) {
            const float4* w4 = reinterpret_cast<const float4*>(sw + (size_t)(nch * KCH + 4 * t4 + s) * NJ);
#pragma unroll
            for (int j = 0; j < NJ / 4; ++j) {
                const float4 ww = w4[j];
                acc[4 * j] = fmaf(av[s], ww.x, acc[4 * j]);
                acc[4 * j + 1] = fmaf(av[s], ww.y, acc[4 * j + 1]);
                acc[4 * j + 2] = fmaf(av[s], ww.z, acc[4 * j + 2]);
                acc[4 * j + 3] = fmaf(av[s], ww.w, acc[4 * j + 3]);
            }
        }
    }
    float* o = static_cast<float*>(g.out) + row * g.n + j0;
    const float* b = g.epilogue == 1 ? static_cast<const float*>(g.bias) + j0 : nullptr;
    const float sc = g.epilogue == 2 ? (float)g.row_scale[row] : 1.f;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        if (j >= (int)nj) break;
        float v = acc[j];
        if (g.epilogue == 1) {
            v += b[j];
            v = v > 0.f ? v : 0.f;
        } else if (g.epilogue == 2) {
            v *= sc;
        }
        acc[j] = v;
    }
    if (nj == (uint32_t)NJ && g.n % 4 == 0 && ((uintptr_t)o % 16 == 0)) {
#pragma unroll
        for (int j = 0; j < NJ; j += 4)
            *reinterpret_cast<float4*>(o + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
    } else {
#pragma unroll
        for (int j = 0; j < NJ; ++j)
            if (j < (int)nj) o[j] = acc[j];
    }
}

// X·W, software-pipelined: 256 rows per CTA (one output row per thread), A
// streamed in 16-column chunks through a double-buffered shared tile (row
// stride 17: conflict-free column reads), the next chunk's four float4 loads
// per thread in flight while the current chunk is consumed, W resident in
// shared memory for the whole kernel (float4 broadcasts).  One barrier per
// chunk.  Requires k % 4 == 0 and a 16-byte aligned A.
constexpr int PR = 256;  // rows per CTA
constexpr int PK = 16;   // k chunk

template <int NJ>
__global__ void __launch_bounds__(PR) k6_gemm_pipe(GemmArgs g) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* sw = reinterpret_cast<float*>(smem_raw);                 // [k][NJ]
    float (*sa)[PR][PK + 1] = reinterpret_cast<float (*)[PR][PK + 1]>(sw + (size_t)g.k * NJ);  // [2][PR][PK+1]
    const float* __restrict__ w = static_cast<const float*>(g.w);
    const float* __restrict__ a = static_cast<const float*>(g.a);
    const uint32_t j0 = blockIdx.y * NJ;
    const uint32_t nj = g.n - j0 < (uint32_t)NJ ? g.n - j0 : (uint32_t)NJ;
    const uint32_t t = threadIdx.x;
    const uint64_t row0 = (uint64_t)blockIdx.x * PR;
    for (uint32_t e = t; e < g.k * NJ; e += PR) {
        const uint32_t r = e / NJ, c = e % NJ;
        sw[e] = c < nj ? __ldg(w + (uint64_t)r * g.n + j0 + c) : 0.f;
    }
    // thread t stages float4 #(t + i*PR) of the [PR][PK] chunk: row (t+i*PR)/4, col4 (t%4)
    constexpr int LPT = PR * PK / 4 / PR;  // float4 loads per thread per chunk (4)
    float4 v[LPT];
    auto load = [&](uint32_t k0) {
#pragma unroll
        for (int i = 0; i < LPT; ++i) {
            const uint32_t e = t + i * PR;
            const uint32_t r = e / (PK / 4), c4 = e % (PK / 4);
            const uint64_t gr = row0 + r;
            const uint32_t kk = k0 + c4 * 4;
            v[i] = (gr < g.m && kk < g.k) ? __ldg(reinterpret_cast<const float4*>(a + gr * g.k + kk))
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int i = 0; i < LPT; ++i) {
            const uint32_t e = t + i * PR;
            const uint32_t r = e / (PK / 4), c = (e % (PK / 4)) * 4;
            sa[buf][r][c] = v[i].x;
            sa[buf][r][c + 1] = v[i].y;
            sa[buf][r][c + 2] = v[i].z;
            sa[buf][r][c + 3] = v[i].w;
        }
    };
    float acc[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[j] = 0.f;
    const uint32_t nch = (g.k + PK - 1) / PK;
    load(0);
    store(0);
    __syncthreads();
    for (uint32_t ch = 0; ch < nch; ++ch) {
        const int buf = ch & 1;
        if (ch + 1 < nch) load((ch + 1) * PK);  // in flight during the FMAs below
        const float* swc = sw + (size_t)ch * PK * NJ;
        const uint32_t kc = g.k - ch * PK < (uint32_t)PK ? g.k - ch * PK : (uint32_t)PK;
        if (kc == (uint32_t)PK) {
#pragma unroll
            for (int kk = 0; kk < PK; ++kk) {
                const float av = sa[buf][t][kk];
#pragma unroll
                for (int j = 0; j < NJ; j += 4) {
                    const float4 ww = *reinterpret_cast<const float4*>(swc + kk * NJ + j);
                    acc[j] = fmaf(av, ww.x, acc[j]);
                    acc[j + 1] = fmaf(av, ww.y, acc[j + 1]);
                    acc[j + 2] = fmaf(av, ww.z, acc[j + 2]);
                    acc[j + 3] = fmaf(av, ww.w, acc[j + 3]);
                }
            }
        } else {
            for (uint32_t kk = 0; kk < kc; ++kk) {
                const float av = sa[buf][t][kk];
#pragma unroll
                for (int j = 0; j < NJ; j += 4) {
                    const float4 ww = *reinterpret_cast<const float4*>(swc + kk * NJ + j);
                    acc[j] = fmaf(av, ww.x, acc[j]);
                    acc[j + 1] = fmaf(av, ww.y, acc[j + 1]);
                    acc[j + 2] = fmaf(av, ww.z, acc[j + 2]);
                    acc[j + 3] = fmaf(av, ww.w, acc[j + 3]);
                }
            }
        }
        if (ch + 1 < nch) store(buf ^ 1);  // the other buffer: last read before the previous barrier
        __syncthreads();
    }
    const uint64_t row = row0 + t;
    if (row >= g.m) return;
    float* o = static_cast<float*>(g.out) + row * g.n + j0;
    const float* bias = g.epilogue == 1 ? static_cast<const float*>(g.bias) + j0 : nullptr;
    const float sc = g.epilogue == 2 ? (float)g.row_scale[row] : 1.f;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        float x = acc[j];
        if (g.epilogue == 1) {
            x += j < (int)nj ? bias[j] : 0.f;
            x = x > 0.f ? x : 0.f;
        } else if (g.epilogue == 2) {
            x *= sc;
        }
        acc[j] = x;
    }
    if (nj == (uint32_t)NJ && g.n % 4 == 0 && ((uintptr_t)o % 16 == 0)) {
#pragma unroll
        for (int j = 0; j < NJ; j += 4)
            *reinterpret_cast<float4*>(o + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
    } else {
#pragma unroll
        for (int j = 0; j < NJ; ++j)
            if (j < (int)nj) o[j] = acc[j];
    }
}

// dW partial = A^T B over a CTA's rows, warp-cooperative: lane l owns rows
// i = l + 32*s (s < PP) of the p-dimension and all QB (padded q) columns;
// per A row a lane loads PP scalars (the warp reads the row coalesced) and
// the B row as QB/4 float4 broadcasts.  The CTA's 8 warp partials are summed
// in warp order in shared memory: one partial per CTA, reduced later in
// chunk order (deterministic).
template <int PP, int QB>
__global__ void __launch_bounds__(256) k6_gemm_tn_warp(const float* __restrict__ a, const float* __restrict__ b,
                                                       uint32_t m, uint32_t p, uint32_t q, uint32_t rows_per_cta,
                                                       float* __restrict__ part) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* red = reinterpret_cast<float*>(smem_raw);  // [8][p*q]
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x / 32;
    const uint64_t r_begin = (uint64_t)blockIdx.x * rows_per_cta;
    const uint64_t r_end = r_begin + rows_per_cta < m ? r_begin + rows_per_cta : m;
    float acc[PP][QB];
#pragma unroll
    for (int s = 0; s < PP; ++s)
#pragma unroll
        for (int j = 0; j < QB; ++j) acc[s][j] = 0.f;
    const bool bvec = (q % 4 == 0) && ((uintptr_t)b % 16 == 0);
#pragma unroll 4
    for (uint64_t r = r_begin + wid; r < r_end; r += 8) {
        float av[PP];
#pragma unroll
        for (int s = 0; s < PP; ++s) {
            const uint32_t i = lane + 32 * s;
            av[s] = i < p ? __ldg(a + r * p + i) : 0.f;
        }
        float bv[QB];
        if (bvec) {
#pragma unroll
            for (int j = 0; j < QB; j += 4) {
                const float4 t = j < (int)q ? __ldg(reinterpret_cast<const float4*>(b + r * q + j))
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
                bv[j] = t.x;
                bv[j + 1] = t.y;
                bv[j + 2] = t.z;
                bv[j + 3] = t.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < QB; ++j) bv[j] = j < (int)q ? __ldg(b + r * q + j) : 0.f;
        }
#pragma unroll
        for (int s = 0; s < PP; ++s)
#pragma unroll
            for (int j = 0; j < QB; ++j) acc[s][j] = fmaf(av[s], bv[j], acc[s][j]);
    }
    // warp partials -> shared memory -> sum over warps in order
#pragma unroll
    for (int s = 0; s < PP; ++s) {
        const uint32_t i = lane + 32 * s;
        if (i < p)
#pragma unroll
            for (int j = 0; j < QB; ++j)
                if (j < (int)q) red[(size_t)wid * p * q + i * q + j] = acc[s][j];
    }
    __syncthreads();
    const uint32_t total = p * q;
    for (uint32_t o = threadIdx.x; o < total; o += blockDim.x) {
        float sum = 0.f;
        for (uint32_t w2 = 0; w2 < 8; ++w2) sum += red[(size_t)w2 * total + o];
        part[(size_t)blockIdx.x * total + o] = sum;
    }
}

// Partial C = A^T B over a chunk of rows, 4x4 register blocks per thread:
// thread (ti, tj) owns C[4ti..4ti+3][4tj..4tj+3]; rows staged 32 at a time
// (float4, 16-byte aligned row strides).  Requires p, q multiples of 4 and
// (p/4)(q/4) <= 1024.
// dW = A^T B for small p*q with any p, q (the widths the tcgen05 path cannot
// TMA, e.g. the 22-class output).  A CTA streams its row range in BK-row
// blocks: each block of A (BK*p floats) and B (BK*q floats) is one contiguous
// run in HBM, copied with 4-byte cp.async (coalesced, no alignment needs)
// into a double-buffered shared tile while the previous block is consumed.
// Thread = one TI x TJ output tile x one row group (rows k = grp mod rg of
// each block); groups are summed in order in shared memory, CTA partials in
// CTA order by the reduce kernel: deterministic.
constexpr int TS_BK = 128;

__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}

template <int TI, int TJ>
__global__ void __launch_bounds__(256) k6_gemm_tn_small(const float* __restrict__ a, const float* __restrict__ b,
                                                        uint32_t m, uint32_t p, uint32_t q, uint32_t rows_per_cta,
                                                        float* __restrict__ part) {
    extern __shared__ __align__(16) float sm[];
    float* sa = sm;                          // [2][TS_BK * p]
    float* sb = sm + 2 * TS_BK * p;          // [2][TS_BK * q]
    const uint32_t tq = (q + TJ - 1) / TJ, tiles = ((p + TI - 1) / TI) * tq;
    const uint32_t rg = blockDim.x / tiles;  // row groups (>= 1: checked by the host)
    const uint32_t t = threadIdx.x, grp = t / tiles, tile = t % tiles;
    const bool active = grp < rg;
    const uint32_t ti = (tile / tq) * TI, tj = (tile % tq) * TJ;
    // vector shared reads of the staged rows (stage bases are 16-byte aligned:
    // sb starts 2·TS_BK·p floats in, each buffer is TS_BK rows long)
    const bool va4 = p % 4 == 0, vb2 = q % 2 == 0;
    const uint64_t r_begin = (uint64_t)blockIdx.x * rows_per_cta;
    const uint64_t r_end = r_begin + rows_per_cta < m ? r_begin + rows_per_cta : m;
    const uint32_t nblk = r_end > r_begin ? (uint32_t)((r_end - r_begin + TS_BK - 1) / TS_BK) : 0u;
    // one contiguous run of floats: 16-byte cp.async where both ends are
    // 16-byte aligned (shared tiles are), 4-byte for the head/tail remainder
    auto copy_run = [&](float* dst, const float* src, uint32_t cnt) {
        const uint32_t head = (uint32_t)((16 - ((uintptr_t)src & 15)) & 15) / 4;
        const bool v16 = (((uintptr_t)src ^ (uintptr_t)dst) & 15) == 0 && cnt > head;
        const uint32_t h = v16 ? head : cnt;
        for (uint32_t e = t; e < h; e += blockDim.x) cp_async4(dst + e, src + e);
        if (!v16) return;
        const uint32_t nv = (cnt - h) / 4;
        for (uint32_t e = t; e < nv; e += blockDim.x)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(dst + h + 4 * e)),
                         "l"(src + h + 4 * e)
                         : "memory");
        for (uint32_t e = h + 4 * nv + t; e < cnt; e += blockDim.x) cp_async4(dst + e, src + e);
    };
    auto load = [&](uint32_t blk, uint32_t buf) {
        const uint64_t r0 = r_begin + (uint64_t)blk * TS_BK;
        const uint32_t nr = (uint32_t)(r_end - r0 < (uint64_t)TS_BK ? r_end - r0 : (uint64_t)TS_BK);
        const float* ga = a + r0 * p;
        const float* gb = b + r0 * q;
        float* da = sa + (size_t)buf * TS_BK * p;
        float* db = sb + (size_t)buf * TS_BK * q;
        copy_run(da, ga, nr * p);
        copy_run(db, gb, nr * q);
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    float acc[TI][TJ];
#pragma unroll
    for (int i = 0; i < TI; ++i)
#pragma unroll
        for (int j = 0; j < TJ; ++j) acc[i][j] = 0.f;
    if (nblk) load(0, 0);
    for (uint32_t blk = 0; blk < nblk; ++blk) {
        const uint32_t buf = blk & 1u;
        if (blk + 1 < nblk) {
            load(blk + 1, buf ^ 1u);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const uint64_t r0 = r_begin + (uint64_t)blk * TS_BK;
        const uint32_t nr = (uint32_t)(r_end - r0 < (uint64_t)TS_BK ? r_end - r0 : (uint64_t)TS_BK);
        if (active) {
            const float* xa = sa + (size_t)buf * TS_BK * p;
            const float* xb = sb + (size_t)buf * TS_BK * q;
#pragma unroll 4
            for (uint32_t k = grp; k < nr; k += rg) {
                float av[TI], bv[TJ];
                if (TI == 4 && va4) {  // p % 4 == 0: one 16-byte shared load
                    const float4 x4 = *reinterpret_cast<const float4*>(xa + k * p + ti);
                    av[0] = x4.x, av[1] = x4.y, av[2] = x4.z, av[3] = x4.w;
                } else {
#pragma unroll
                    for (int i = 0; i < TI; ++i) av[i] = ti + i < p ? xa[k * p + ti + i] : 0.f;
                }
                if (TJ % 2 == 0 && vb2) {  // q even: 8-byte shared loads, pairs wholly in or out
#pragma unroll
                    for (int j = 0; j < TJ; j += 2) {
                        const float2 y2 = tj + j < q ? *reinterpret_cast<const float2*>(xb + k * q + tj + j)
                                                     : make_float2(0.f, 0.f);
                        bv[j] = y2.x, bv[j + 1] = y2.y;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < TJ; ++j) bv[j] = tj + j < q ? xb[k * q + tj + j] : 0.f;
                }
#pragma unroll
                for (int i = 0; i < TI; ++i)
#pragma unroll
                    for (int j = 0; j < TJ; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
            }
        }
        __syncthreads();  // the buffer is refilled by the next iteration's load
    }
    // row groups -> shared memory (the staging area is free) -> sum in group order
    float* red = sm;  // [rg][p*q]
    const uint32_t total = p * q;
    if (active)
#pragma unroll
        for (int i = 0; i < TI; ++i)
#pragma unroll
            for (int j = 0; j < TJ; ++j)
                if (ti + i < p && tj + j < q) red[(size_t)grp * total + (ti + i) * q + tj + j] = acc[i][j];
    __syncthreads();
    for (uint32_t o = t; o < total; o += blockDim.x) {
        float sum = 0.f;
        for (uint32_t g2 = 0; g2 < rg; ++g2) sum += red[(size_t)g2 * total + o];
        part[(size_t)blockIdx.x * total + o] = sum;
    }
}

// ------------------------------------------------- K6 dense backward (fused)
// Backward of the node update y = z W (matmul, engine.cpp:315-331) in one
// pass over the rows, for the narrow widths of the GCN output layer (C3:
// z 16 wide, y 22 wide, whose 88-byte rows no TMA descriptor can stride):
//   dz = row_scale ⊙ (dy Wᵀ)          (m x p)
//   dW = zᵀ dy                         (p x q, per-CTA partials summed in
//                                       CTA order by k_reduce_partials)
// Both read dy; one kernel reads dy and z once instead of the two passes of
// k6_gemm_flat + k6_gemm_tn_small.  A CTA owns a contiguous row chunk
// (deterministic partials) and streams it in DB_ROWS-row tiles with a
// double-buffered cp.async pipeline (the same copy_run scheme as
// k6_gemm_tn_small).  dz: 4 threads per row, each 4 output columns (W held
// k-major in shared memory, one 16-byte broadcast read per k), stored as
// one coalesced float4 per thread.  dW: TI x TJ = 4 x 4 register tiles over
// row groups, summed in group order at the end.
#ifndef GNNA_DB_ROWS
#define GNNA_DB_ROWS 64
#endif
#ifndef GNNA_DB_STAGES
#define GNNA_DB_STAGES 4
#endif
constexpr int DB_ROWS = GNNA_DB_ROWS, DB_STAGES = GNNA_DB_STAGES, DB_P = 32, DB_Q = 32;

// Compile-time widths (P, Q <= 32): every inner loop unrolls, operands are
// read as 16-/8-byte shared vectors and the FMA chains are independent.
// Warp roles: warps 0-3 compute dz (one row half per thread per tile), warps
// 4-7 accumulate dW (their 4x8 register tiles stay live only on that side,
// so the kernel's register count is the larger role's, not the sum: 4 CTAs
// of 256 threads per SM).  Both roles run the same tile loop and meet at
// the same CTA barriers; all 256 threads issue the cp.async ring.
template <int P, int Q>
__global__ void __launch_bounds__(256, 4) k6_dense_bwd(const float* __restrict__ dy, const float* __restrict__ w,
                                                    const float* __restrict__ z, const double* __restrict__ row_scale,
                                                    uint32_t m, uint32_t rows_per_cta, float* __restrict__ dz,
                                                    float* __restrict__ part) {
    static_assert(P % 4 == 0 && Q % 2 == 0 && P <= DB_P && Q <= DB_Q, "dense_bwd widths");
    constexpr int TI = 4, TJ = 8;                       // dW register tile
    constexpr int TQ = (Q + TJ - 1) / TJ, TILES = (P / TI) * TQ, RG = 128 / TILES;
    constexpr int PH = P / 2;                           // dz: 2 threads per row, PH outputs each
    static_assert(2 * DB_ROWS % 128 == 0 && RG >= 1, "dense_bwd tiling");
    extern __shared__ __align__(16) float sm[];
    float* sdy = sm;                                    // [S][DB_ROWS * Q]
    float* sz = sdy + DB_STAGES * DB_ROWS * Q;          // [S][DB_ROWS * P]
    float* swt = sz + DB_STAGES * DB_ROWS * P;          // [Q][P]: W^T, k-major
    double* srs = reinterpret_cast<double*>(swt + Q * P + (Q * P) % 2);  // [S][DB_ROWS] row scales
    const uint32_t t = threadIdx.x;
    for (uint32_t e = t; e < Q * P; e += blockDim.x) {
        const uint32_t k = e / P, i = e % P;
        swt[e] = __ldg(w + (size_t)i * Q + k);
    }
    const uint64_t r_begin = (uint64_t)blockIdx.x * rows_per_cta;
    const uint64_t r_end = r_begin + rows_per_cta < m ? r_begin + rows_per_cta : m;
    const uint32_t nblk = r_end > r_begin ? (uint32_t)((r_end - r_begin + DB_ROWS - 1) / DB_ROWS) : 0u;
    auto copy_run = [&](float* dst, const float* src, uint32_t cnt) {
        const uint32_t head = (uint32_t)((16 - ((uintptr_t)src & 15)) & 15) / 4;
        const bool v16 = (((uintptr_t)src ^ (uintptr_t)dst) & 15) == 0 && cnt > head;
        const uint32_t h = v16 ? head : cnt;
        for (uint32_t e = t; e < h; e += blockDim.x) cp_async4(dst + e, src + e);
        if (!v16) return;
        const uint32_t nv = (cnt - h) / 4;
        for (uint32_t e = t; e < nv; e += blockDim.x)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(dst + h + 4 * e)),
                         "l"(src + h + 4 * e)
                         : "memory");
        for (uint32_t e = h + 4 * nv + t; e < cnt; e += blockDim.x) cp_async4(dst + e, src + e);
    };
    // one commit group per ring slot (empty past the chunk, so wait_group counts stay uniform)
    auto load = [&](uint32_t blk) {
        if (blk < nblk) {
            const uint32_t buf = blk % DB_STAGES;
            const uint64_t r0 = r_begin + (uint64_t)blk * DB_ROWS;
            const uint32_t nr = (uint32_t)(r_end - r0 < (uint64_t)DB_ROWS ? r_end - r0 : (uint64_t)DB_ROWS);
            copy_run(sdy + (size_t)buf * DB_ROWS * Q, dy + r0 * Q, nr * Q);
            copy_run(sz + (size_t)buf * DB_ROWS * P, z + r0 * P, nr * P);
            if (row_scale)
                for (uint32_t e = t; e < nr; e += blockDim.x)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                                     (uint32_t)__cvta_generic_to_shared(srs + (size_t)buf * DB_ROWS + e)),
                                 "l"(row_scale + r0 + e)
                                 : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // the tile loop both roles run: wait for tile blk, work(blk), free its slot
    auto pipeline = [&](auto&& work) {
#pragma unroll
        for (int s = 0; s < DB_STAGES - 1; ++s) load(s);
        for (uint32_t blk = 0; blk < nblk; ++blk) {
            load(blk + DB_STAGES - 1);  // refills the slot freed at the end of the previous iteration
            asm volatile("cp.async.wait_group %0;" ::"n"(DB_STAGES - 1) : "memory");
            asm volatile("barrier.sync 1, 256;" ::: "memory");  // non-.aligned: the roles reach it from different code
            const uint32_t buf = blk % DB_STAGES;
            const uint64_t r0 = r_begin + (uint64_t)blk * DB_ROWS;
            const uint32_t nr = (uint32_t)(r_end - r0 < (uint64_t)DB_ROWS ? r_end - r0 : (uint64_t)DB_ROWS);
            work(buf, r0, nr, sdy + (size_t)buf * DB_ROWS * Q, sz + (size_t)buf * DB_ROWS * P);
            asm volatile("barrier.sync 1, 256;" ::: "memory");  // non-.aligned: the roles reach it from different code  // slot `buf` is refilled next iteration
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    };
    float* red = sm;  // [RG][P*Q] after the loop (the staging area is free)
    constexpr uint32_t total = P * Q;
    if (t < 128) {
        // dz = row_scale * (dy W^T): 2 threads per row, PH outputs each
        pipeline([&](uint32_t buf, uint64_t r0, uint32_t nr, const float* xdy, const float*) {
            for (uint32_t it = t; it < 2 * DB_ROWS; it += 128) {
                const uint32_t dr = it / 2, half = it % 2;
                if (dr >= nr) break;
                float yv[Q];
#pragma unroll
                for (int k = 0; k < Q; k += 2) {
                    const float2 y2 = *reinterpret_cast<const float2*>(xdy + dr * Q + k);
                    yv[k] = y2.x;
                    yv[k + 1] = y2.y;
                }
                // packed FFMA2 (two lanes of one fma.rn each: the same roundings as scalar fmaf)
                float2 o[PH / 2];
#pragma unroll
                for (int c = 0; c < PH / 2; ++c) o[c] = make_float2(0.f, 0.f);
#pragma unroll
                for (int k = 0; k < Q; ++k) {
                    const float2 yk = make_float2(yv[k], yv[k]);
#pragma unroll
                    for (int c = 0; c < PH; c += 4) {
                        const float4 w4 = *reinterpret_cast<const float4*>(swt + k * P + half * PH + c);
                        o[c / 2] = __ffma2_rn(yk, make_float2(w4.x, w4.y), o[c / 2]);
                        o[c / 2 + 1] = __ffma2_rn(yk, make_float2(w4.z, w4.w), o[c / 2 + 1]);
                    }
                }
                const float s = row_scale ? (float)srs[(size_t)buf * DB_ROWS + dr] : 1.f;
                float4* out = reinterpret_cast<float4*>(dz + (r0 + dr) * P + half * PH);
#pragma unroll
                for (int c = 0; c < PH; c += 4)
                    out[c / 4] = make_float4(s * o[c / 2].x, s * o[c / 2].y, s * o[c / 2 + 1].x, s * o[c / 2 + 1].y);
            }
        });
        asm volatile("barrier.sync 1, 256;" ::: "memory");  // non-.aligned: the roles reach it from different code  // the dW side writes its partials into `red`
        asm volatile("barrier.sync 1, 256;" ::: "memory");  // non-.aligned: the roles reach it from different code
    } else {
        // dW += z^T dy (TI x TJ register tile per thread, RG row groups)
        const uint32_t td = t - 128, grp = td / TILES, tile = td % TILES;
        const bool active = grp < RG;
        const uint32_t ti = (tile / TQ) * TI, tj = (tile % TQ) * TJ;
        float2 acc[TI][TJ / 2];  // column pairs: packed FFMA2
#pragma unroll
        for (int i = 0; i < TI; ++i)
#pragma unroll
            for (int j = 0; j < TJ / 2; ++j) acc[i][j] = make_float2(0.f, 0.f);
        pipeline([&](uint32_t, uint64_t, uint32_t nr, const float* xdy, const float* xz) {
            if (!active) return;
            for (uint32_t k = grp; k < nr; k += RG) {
                const float4 a4 = *reinterpret_cast<const float4*>(xz + k * P + ti);
                float2 bv[TJ / 2];
#pragma unroll
                for (int j = 0; j < TJ; j += 2)
                    bv[j / 2] = tj + j < Q ? *reinterpret_cast<const float2*>(xdy + k * Q + tj + j)
                                           : make_float2(0.f, 0.f);
                const float av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
                for (int i = 0; i < TI; ++i)
#pragma unroll
                    for (int j = 0; j < TJ / 2; ++j)
                        acc[i][j] = __ffma2_rn(make_float2(av[i], av[i]), bv[j], acc[i][j]);
            }
        });
        asm volatile("barrier.sync 1, 256;" ::: "memory");  // non-.aligned: the roles reach it from different code  // every role is out of the ring
        if (active)
#pragma unroll
            for (int i = 0; i < TI; ++i)
#pragma unroll
                for (int j = 0; j < TJ; ++j)
                    if (tj + j < Q)
                        red[(size_t)grp * total + (ti + i) * Q + tj + j] = j % 2 ? acc[i][j / 2].y : acc[i][j / 2].x;
        asm volatile("barrier.sync 1, 256;" ::: "memory");  // non-.aligned: the roles reach it from different code
    }
    for (uint32_t o = t; o < total; o += blockDim.x) {
        float sum = 0.f;
        for (uint32_t g2 = 0; g2 < RG; ++g2) sum += red[(size_t)g2 * total + o];
        part[(size_t)blockIdx.x * total + o] = sum;
    }
}

template <int P, int Q>
void launch_dense_bwd(gnna_ctx* ctx, const float* dy, const float* w, const float* z, const double* rs, uint32_t m,
                      float* dz, float* dw) {
    constexpr int TQ = (Q + 7) / 8, TILES = (P / 4) * TQ, RG = 128 / TILES;
    const size_t sbytes = std::max<size_t>((size_t)(DB_STAGES * DB_ROWS * (P + Q) + Q * P + (Q * P) % 2 +
                                                    2 * DB_STAGES * DB_ROWS),
                                           (size_t)RG * P * Q) * 4;
    static int occ = -1;
    if (occ < 0) {
        GNNA_CUDA(cudaFuncSetAttribute(k6_dense_bwd<P, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sbytes));
        GNNA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k6_dense_bwd<P, Q>, 256, sbytes));
        occ = std::max(occ, 1);
    }
    uint32_t ctas = std::max<uint32_t>(1, std::min<uint32_t>((uint32_t)occ * ctx->num_sms, (m + DB_ROWS - 1) / DB_ROWS));
    const uint32_t rpc = ((m + ctas - 1) / ctas + DB_ROWS - 1) / DB_ROWS * DB_ROWS;
    ctas = (m + rpc - 1) / rpc;
    gnna::DevBuf<float> part((size_t)ctas * P * Q, ctx->stream);
    k6_dense_bwd<P, Q><<<ctas, 256, sbytes, ctx->stream>>>(dy, w, z, rs, m, rpc, dz, part.get());
    gnna::launched(ctx, "k6_dense_bwd");
    gnna::reduce_partials(ctx, part.get(), ctas, P * Q, dw);
}

constexpr int TN4_ROWS = 32;

__global__ void k6_gemm_tn4(const float* __restrict__ a, const float* __restrict__ b, uint32_t m, uint32_t p,
                            uint32_t q, uint32_t rows_per_chunk, float* __restrict__ part) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float4* sa = reinterpret_cast<float4*>(smem_raw);  // [TN4_ROWS][p/4]
    float4* sb = sa + (size_t)TN4_ROWS * (p / 4);     // [TN4_ROWS][q/4]
    const uint32_t p4 = p / 4, q4 = q / 4;
    const uint32_t ti = threadIdx.x / q4, tj = threadIdx.x % q4;
    const uint64_t r_begin = (uint64_t)blockIdx.x * rows_per_chunk;
    const uint64_t r_end = r_begin + rows_per_chunk < m ? r_begin + rows_per_chunk : m;
    float acc[4][4] = {};
    const float4* a4 = reinterpret_cast<const float4*>(a);
    const float4* b4 = reinterpret_cast<const float4*>(b);
    for (uint64_t r0 = r_begin; r0 < r_end; r0 += TN4_ROWS) {
        const uint32_t nr = (uint32_t)(r_end - r0 < (uint64_t)TN4_ROWS ? r_end - r0 : (uint64_t)TN4_ROWS);
#pragma unroll 8
        for (uint32_t e = threadIdx.x; e < TN4_ROWS * p4; e += blockDim.x) {
            const uint32_t r = e / p4;
            sa[e] = r < nr ? __ldg(a4 + (r0 + r) * p4 + e % p4) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll 4
        for (uint32_t e = threadIdx.x; e < TN4_ROWS * q4; e += blockDim.x) {
            const uint32_t r = e / q4;
            sb[e] = r < nr ? __ldg(b4 + (r0 + r) * q4 + e % q4) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncthreads();
        if (ti < p4) {
            for (uint32_t r = 0; r < nr; ++r) {
                const float4 x = sa[r * p4 + ti], y = sb[r * q4 + tj];
                const float xa[4] = {x.x, x.y, x.z, x.w}, ya[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(xa[i], ya[j], acc[i][j]);
            }
        }
        __syncthreads();
    }
    if (ti >= p4) return;
    float* out = part + (size_t)blockIdx.x * p * q;
#pragma unroll
    for (int i = 0; i < 4; ++i)
        *reinterpret_cast<float4*>(out + (size_t)(4 * ti + i) * q + 4 * tj) =
            make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
}

// Deterministic chunk reduction with a warp per output: lanes take chunks
// lane, lane+32, ... and a fixed shuffle tree combines them.
__global__ void k6_reduce_chunks_warp(const float* __restrict__ part, uint32_t chunks, uint32_t total,
                                      float* __restrict__ out) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t o = blockIdx.x * (uint64_t)(blockDim.x / 32) + threadIdx.x / 32; o < total; o += warps) {
        float s = 0.f;
        for (uint32_t c = lane; c < chunks; c += 32) s += part[(size_t)c * total + o];
        for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) out[o] = s;
    }
}

template <class T>
void launch_gemm(gnna_ctx* ctx, const GemmArgs& g, bool exact) {
    if (g.m == 0 || g.n == 0) return;
    if constexpr (std::is_same<T, float>::value) {
        if (!exact) {
            static const bool no_flat = std::getenv("GNNA_GEMM_NOFLAT") != nullptr;  // A/B switches
            static const bool all_flat = std::getenv("GNNA_GEMM_FLAT") != nullptr;
            // Only where the tcgen05 path cannot TMA-tile A (k % 4 != 0): in the
            // C3 train step the 22 -> 16 product takes 25.1 us here against 41.0
            // on tcgen05 with scalar A loads, while 16 -> 22 stays on TMA (22.9
            // us, flat 24.2; ncu, profiles/r01p_gemm_flat.md).
            if (!no_flat && g.k <= (uint32_t)FL_K && g.n <= (uint32_t)FL_K && (g.k % 4 != 0 || all_flat) &&
                (uintptr_t)g.a % 16 == 0 && (uintptr_t)g.out % 16 == 0) {
                static const int per_sm = std::getenv("GNNA_FLAT_CTAS") ? std::atoi(std::getenv("GNNA_FLAT_CTAS")) : 4;
                const uint64_t tiles = (g.m + FL_ROWS - 1) / FL_ROWS;
                const dim3 grid((unsigned)std::min<uint64_t>(tiles, (uint64_t)per_sm * ctx->num_sms));
                if (g.n <= 8)
                    k6_gemm_flat<8><<<grid, FL_ROWS, 0, ctx->stream>>>(g);
                else if (g.n <= 16)
                    k6_gemm_flat<16><<<grid, FL_ROWS, 0, ctx->stream>>>(g);
                else if (g.n <= 24)
                    k6_gemm_flat<24><<<grid, FL_ROWS, 0, ctx->stream>>>(g);
                else
                    k6_gemm_flat<32><<<grid, FL_ROWS, 0, ctx->stream>>>(g);
                gnna::launched(ctx, "k6_gemm_flat");
                return;
            }
            static const bool simt = std::getenv("GNNA_GEMM_SIMT") != nullptr;  // A/B switch
            if (!simt && gnna::gemm_tc_f32(ctx, static_cast<const float*>(g.a), static_cast<const float*>(g.w),
                                           static_cast<const float*>(g.bias), g.row_scale, static_cast<float*>(g.out),
                                           g.m, g.k, g.n, g.epilogue))
                return;
            const uint32_t nj = g.n <= 4 ? 4 : g.n <= 8 ? 8 : g.n <= 16 ? 16 : 32;
            dim3 grid((g.m + ROWS - 1) / ROWS, (g.n + nj - 1) / nj);
            const size_t wbytes = (size_t)g.k * nj * 4;
            const size_t pbytes = wbytes + (size_t)2 * PR * (PK + 1) * 4;
            static const bool use_rows = std::getenv("GNNA_GEMM_ROWS") != nullptr;  // A/B switch
            if (!use_rows && g.k % 4 == 0 && ((uintptr_t)g.a % 16 == 0) && pbytes <= 200 * 1024) {
                dim3 pgrid((g.m + PR - 1) / PR, (g.n + nj - 1) / nj);
                auto launch = [&](auto kern) {
                    if (pbytes > 48 * 1024)
                        GNNA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pbytes));
                    kern<<<pgrid, PR, pbytes, ctx->stream>>>(g);
                };
                switch (nj) {
                    case 4: launch(k6_gemm_pipe<4>); break;
                    case 8: launch(k6_gemm_pipe<8>); break;
                    case 16: launch(k6_gemm_pipe<16>); break;
                    default: launch(k6_gemm_pipe<32>); break;
                }
                gnna::launched(ctx, "k6_gemm_pipe");
                return;
            }
            if (g.k % 4 == 0 && ((uintptr_t)g.a % 16 == 0) && wbytes <= 64 * 1024) {
                auto launch = [&](auto kern) {
                    if (wbytes > 48 * 1024)
                        GNNA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wbytes));
                    kern<<<grid, 128, wbytes, ctx->stream>>>(g);
                };
                switch (nj) {
                    case 4: launch(k6_gemm_rows<4>); break;
                    case 8: launch(k6_gemm_rows<8>); break;
                    case 16: launch(k6_gemm_rows<16>); break;
                    default: launch(k6_gemm_rows<32>); break;
                }
                gnna::launched(ctx, "k6_gemm_rows");
                return;
            }
            switch (nj) {
                case 4: k6_gemm_f32<4><<<grid, ROWS, 0, ctx->stream>>>(g); break;
                case 8: k6_gemm_f32<8><<<grid, ROWS, 0, ctx->stream>>>(g); break;
                case 16: k6_gemm_f32<16><<<grid, ROWS, 0, ctx->stream>>>(g); break;
                default: k6_gemm_f32<32><<<grid, ROWS, 0, ctx->stream>>>(g); break;
            }
            gnna::launched(ctx, "k6_gemm_f32");
            return;
        }
    }
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
    if constexpr (std::is_same<T, float>::value) {
        if (gnna::gemm_tn_tc_f32(ctx, a, b, m, p, q, out)) return;
        constexpr uint32_t TI = 4, TJ = 4;
        const uint32_t tiles = ((p + TI - 1) / TI) * ((q + TJ - 1) / TJ);
        const size_t sbytes = std::max<size_t>((size_t)2 * TS_BK * (p + q), (size_t)(256 / std::max(tiles, 1u)) * p * q) * 4;
        static const bool no_small = std::getenv("GNNA_TN_WARP") != nullptr;  // A/B switch
        if (!no_small && tiles <= 256 && sbytes <= 96 * 1024) {
            static const uint32_t per_sm =
                std::getenv("GNNA_TN_SMALL_CTAS") ? (uint32_t)std::atoi(std::getenv("GNNA_TN_SMALL_CTAS")) : 4u;
            uint32_t ctas = std::max<uint32_t>(1, std::min<uint32_t>(per_sm * ctx->num_sms, (m + TS_BK - 1) / TS_BK));
            const uint32_t rpc = ((m + ctas - 1) / ctas + TS_BK - 1) / TS_BK * TS_BK;
            ctas = (m + rpc - 1) / rpc;
            const uint32_t total = p * q;
            DevBuf<float> part((size_t)ctas * total, ctx->stream);
            if (sbytes > 48 * 1024)
                GNNA_CUDA(cudaFuncSetAttribute(k6_gemm_tn_small<TI, TJ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)sbytes));
            k6_gemm_tn_small<TI, TJ><<<ctas, 256, sbytes, ctx->stream>>>(a, b, m, p, q, rpc, part.get());
            gnna::launched(ctx, "k6_gemm_tn_small");
            static const bool seq = std::getenv("GNNA_TN_SEQ_REDUCE") != nullptr;  // A/B switch
            if (seq) {
                k6_reduce_chunks_warp<<<gnna::grid_for((uint64_t)total * 32, 256), 256, 0, ctx->stream>>>(
                    part.get(), ctas, total, out);
                gnna::launched(ctx, "k6_reduce_chunks_warp");
            } else {
                gnna::k_reduce_partials<<<(total + 31) / 32, 1024, 0, ctx->stream>>>(part.get(), ctas, total, out);
                gnna::launched(ctx, "k_reduce_partials");
            }
            return;
        }
        if (p <= 128 && q <= 32) {
            const uint32_t pp = (p + 31) / 32;
            const uint32_t qb = q <= 4 ? 4 : q <= 8 ? 8 : q <= 16 ? 16 : 32;
            uint32_t ctas = std::max<uint32_t>(1, std::min<uint32_t>(2 * ctx->num_sms, (m + 255) / 256));
            const uint32_t rpc = (m + ctas - 1) / ctas;
            ctas = (m + rpc - 1) / rpc;
            DevBuf<float> part((size_t)ctas * total, ctx->stream);
            const size_t smem = (size_t)8 * total * sizeof(float);
            auto launch = [&](auto kern) {
                if (smem > 48 * 1024)
                    GNNA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                kern<<<ctas, 256, smem, ctx->stream>>>(a, b, m, p, q, rpc, part.get());
            };
#define GNNA_TNW(PP)                                           \
    switch (qb) {                                              \
        case 4: launch(k6_gemm_tn_warp<PP, 4>); break;         \
        case 8: launch(k6_gemm_tn_warp<PP, 8>); break;         \
        case 16: launch(k6_gemm_tn_warp<PP, 16>); break;       \
        default: launch(k6_gemm_tn_warp<PP, 32>); break;       \
    }
            switch (pp) {
                case 1: GNNA_TNW(1) break;
                case 2: GNNA_TNW(2) break;
                case 3: GNNA_TNW(3) break;
                default: GNNA_TNW(4) break;
            }
#undef GNNA_TNW
            gnna::launched(ctx, "k6_gemm_tn_warp");
            static const bool seq = std::getenv("GNNA_TN_SEQ_REDUCE") != nullptr;  // A/B switch
            if (seq) {
                k6_reduce_chunks_warp<<<gnna::grid_for((uint64_t)total * 32, 256), 256, 0, ctx->stream>>>(
                    part.get(), ctas, total, out);
                gnna::launched(ctx, "k6_reduce_chunks_warp");
            } else {
                gnna::k_reduce_partials<<<(total + 31) / 32, 1024, 0, ctx->stream>>>(part.get(), ctas, total, out);
                gnna::launched(ctx, "k_reduce_partials");
            }
            return;
        }
        const bool aligned = ((uintptr_t)a % 16 == 0) && ((uintptr_t)b % 16 == 0) && ((uintptr_t)out % 16 == 0);
        if (aligned && p % 4 == 0 && q % 4 == 0 && (p / 4) * (q / 4) <= 1024) {
            const uint32_t threads = ((p / 4) * (q / 4) + 31) / 32 * 32;
            uint32_t chunks = std::max<uint32_t>(1, std::min<uint32_t>(8 * ctx->num_sms, (m + 63) / 64));
            const uint32_t rpc = (m + chunks - 1) / chunks;
            chunks = (m + rpc - 1) / rpc;
            DevBuf<float> part((size_t)chunks * total, ctx->stream);
            const size_t smem = (size_t)TN4_ROWS * (p + q) * sizeof(float);
            if (smem > 48 * 1024)
                GNNA_CUDA(cudaFuncSetAttribute(k6_gemm_tn4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k6_gemm_tn4<<<chunks, threads, smem, ctx->stream>>>(a, b, m, p, q, rpc, part.get());
            gnna::launched(ctx, "k6_gemm_tn4");
            k6_reduce_chunks_warp<<<gnna::grid_for((uint64_t)total * 32, 256), 256, 0, ctx->stream>>>(
                part.get(), chunks, total, out);
            gnna::launched(ctx, "k6_reduce_chunks_warp");
            return;
        }
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

// Backward of y = z W for narrow layers, fused (see k6_dense_bwd):
// dz = row_scale ⊙ (dy Wᵀ) and dW = zᵀ dy in one pass (fp32); the fp64 path
// (and wide layers) runs the two products separately, in the exact orders.
extern "C" gnna_status gnna_dense_backward(gnna_ctx* ctx, int dtype, const void* d_dy, uint32_t m, uint32_t q,
                                           const void* d_w, const void* d_z, uint32_t p, const double* d_row_scale,
                                           void* d_dz, void* d_dw) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (dtype != GNNA_F32 && dtype != GNNA_F64) gnna::raise(GNNA_ERR_DOMAIN, "unknown dtype");
        if (!d_dz || !d_dw) gnna::raise(GNNA_ERR_DOMAIN, "dense_backward: null output");
        const uint32_t total = p * q;
        (void)total;
        static const bool off = std::getenv("GNNA_DENSE_BWD") && std::atoi(std::getenv("GNNA_DENSE_BWD")) == 0;
        if (dtype == GNNA_F32 && !off && m > 0 && (uintptr_t)d_dy % 16 == 0 && (uintptr_t)d_z % 16 == 0 &&
            (uintptr_t)d_dz % 16 == 0) {
            const auto dy = static_cast<const float*>(d_dy);
            const auto w = static_cast<const float*>(d_w);
            const auto z = static_cast<const float*>(d_z);
            auto dz = static_cast<float*>(d_dz);
            auto dw = static_cast<float*>(d_dw);
            // instantiated widths: the GCN output layers of the configs (C3: 16 x 22)
            if (p == 16 && q == 22) return launch_dense_bwd<16, 22>(ctx, dy, w, z, d_row_scale, m, dz, dw);
            if (p == 16 && q == 16) return launch_dense_bwd<16, 16>(ctx, dy, w, z, d_row_scale, m, dz, dw);
            if (p == 16 && q == 8) return launch_dense_bwd<16, 8>(ctx, dy, w, z, d_row_scale, m, dz, dw);
            if (p == 32 && q == 32) return launch_dense_bwd<32, 32>(ctx, dy, w, z, d_row_scale, m, dz, dw);
            if (p == 32 && q == 22) return launch_dense_bwd<32, 22>(ctx, dy, w, z, d_row_scale, m, dz, dw);
        }
        // separate products: dW = z^T dy; dz = dy W^T (W^T materialised), row-scaled
        gnna::gemm_tn(ctx, dtype, d_z, d_dy, m, p, q, d_dw);
        const size_t el = dtype == GNNA_F32 ? 4 : 8;
        gnna::DevBuf<uint8_t> wt((size_t)total * el, ctx->stream);
        gnna::transpose(ctx, dtype, d_w, p, q, wt.get());
        gnna::gemm(ctx, dtype, d_dy, m, q, wt.get(), p, nullptr, d_row_scale ? 2 : 0, d_row_scale, d_dz);
    });
}
