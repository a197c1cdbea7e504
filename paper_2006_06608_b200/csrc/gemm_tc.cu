// K6-TC: the fp32 node update X·W (engine.cpp:315-331 matmul, the fast path
// of gcn_layer / gin_layer) on the 5th-generation tensor cores.
//
// tcgen05.mma kind::tf32 with the 3xTF32 split: every fp32 operand x is
// written to shared memory as hi = rna_tf32(x) and lo = rna_tf32(x - hi), and
// the product is accumulated in TMEM (fp32) as A_hi·W_hi + A_hi·W_lo +
// A_lo·W_hi.  The dropped lo·lo term and the tf32 rounding of lo are ~2^-22
// relative per product, so results stay inside the fp32 parity bar (1e-5 of
// sum|terms|, tests/test_layers_gpu.py) that a plain tf32 MMA would break.
//
// Shape of the work: m = nodes (10^5..10^7) by small k, n (<= 128): HBM-bound
// (C3: 410k x 96 . 96 x 16 moves 184 MB for 1.3 GFLOP).  Two kernels:
//
// k6_gemm_tc_tma (k % 4 == 0, 16-byte aligned A; the common case), persistent,
// one CTA per SM, warp-specialised:
//   * warp 8 issues TMA (cp.async.bulk.tensor, box 32 fp32 x 128 rows per K
//     slice, SWIZZLE_128B) into an S-deep ring of stages and the MMAs;
//   * the TMA'd tile IS the canonical SW128 K-major operand and, read as
//     tf32, IS A_hi (truncated) -- it feeds tcgen05.mma straight from smem
//     against [W_hi ; W_lo] (N = 2*NP: both cross terms in one instruction);
//   * two groups of 4 warps take alternate tiles: each thread (= TMEM lane =
//     tile row) reads its row from the swizzled stage (conflict-free), writes
//     A_lo = x - trunc(x) (lo_part2) into TMEM with tcgen05.st, and the MMA
//     warp runs A_lo x W_hi with A from TMEM; the group then tcgen05.ld's its
//     accumulator, adds the hi/lo column halves, applies the fused epilogue
//     and stores the 32-row run of each warp coalesced via shared memory.
//   Hand-offs are mbarriers only (no CTA-wide barrier in the loop).
//
// k6_gemm_tc (any k <= 128, any alignment): each thread loads its row into
// registers one tile ahead, splits hi/lo into the no-swizzle K-major layout
// (chunk c of row r at c*2048 + r*16: LBO 2048 B, SBO 128 B) and one thread
// issues 3 MMAs per K step.
//
// Padding of k to KP and n to NP is zero-filled on chip only; HBM traffic stays
// at the algorithmic m*(k+n)*4 bytes.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "gnna_common.cuh"

namespace gnna {

namespace {

constexpr int TM = 128;  // rows per tile = MMA M = TMEM lanes

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float rna_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// UMMA shared-memory descriptor, SWIZZLE_NONE, K-major canonical layout
// ((8,m),2):((16B,SBO),LBO); version 1 (sm_100), base offset 0.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// Instruction descriptor kind::tf32: D f32, A/B tf32, both K-major, M=128.
template <int NP>
__device__ __forceinline__ constexpr uint32_t idesc_tf32() {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NP >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    const long long t0 = clock64();
    while (true) {
        uint32_t done;
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
        if (done) return;
        if (clock64() - t0 > (1ll << 34)) __trap();  // ~10 s: never hang the device
    }
}

// 16 consecutive TMEM columns of this warp's 32 lanes -> 16 registers.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

struct TcArgs {
    const float* a;
    const float* w;
    const float* bias;       // epilogue 1
    const double* row_scale;  // epilogue 2
    float* out;
    uint32_t m, k, n;
    int epilogue;  // 0 none, 1 bias + relu, 2 row scale
    uint32_t tiles;
    int vec;   // A rows are float4-loadable (k % 4 == 0, 16-byte aligned)
    int vec2;  // A rows are float2-loadable (k % 2 == 0, 8-byte aligned)
};

template <int KP, int NP>
__global__ void __launch_bounds__(TM) k6_gemm_tc(TcArgs g) {
    static_assert(KP % 8 == 0 && KP <= 128, "KP");
    static_assert(NP % 16 == 0 && NP >= 16 && NP <= 64, "NP");
    constexpr int KC = KP / 4;                  // 16-byte chunks per row
    constexpr uint32_t A_CH = TM * 16;          // bytes per A chunk column (128 rows)
    constexpr uint32_t W_CH = NP * 16;          // bytes per W chunk column (NP rows)
    constexpr uint32_t A_BYTES = KC * A_CH;
    constexpr uint32_t W_BYTES = KC * W_CH;
    constexpr uint32_t TCOLS = NP < 32 ? 32 : NP;  // TMEM allocation: power of two >= 32
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* s_ahi = smem;
    unsigned char* s_alo = smem + A_BYTES;
    unsigned char* s_whi = smem + 2 * A_BYTES;
    unsigned char* s_wlo = smem + 2 * A_BYTES + W_BYTES;
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_slot;

    const uint32_t t = threadIdx.x, warp = t / 32, lane = t % 32;
    const uint32_t j0 = blockIdx.y * NP;
    const uint32_t nj = g.n - j0 < (uint32_t)NP ? g.n - j0 : (uint32_t)NP;

    // W^T block (NP x KP, K-major), split once per CTA
    for (uint32_t e = t; e < (uint32_t)(NP * KP); e += TM) {
        const uint32_t nn = e / KP, kk = e % KP;
        const float x = (nn < nj && kk < g.k) ? __ldg(g.w + (uint64_t)kk * g.n + j0 + nn) : 0.f;
        const float hi = rna_tf32(x), lo = rna_tf32(x - hi);
        const uint32_t off = (kk / 4) * W_CH + nn * 16 + (kk % 4) * 4;
        *reinterpret_cast<float*>(s_whi + off) = hi;
        *reinterpret_cast<float*>(s_wlo + off) = lo;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                     "r"(TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_slot;
    const uint32_t bar_a = smem_u32(&bar);

    float4 v[KC];  // this thread's row of the tile being loaded
    auto load = [&](uint32_t tile) {
        const uint64_t row = (uint64_t)tile * TM + t;
        if (g.vec) {
            const float4* src = reinterpret_cast<const float4*>(g.a + row * g.k);
#pragma unroll
            for (int c = 0; c < KC; ++c)
                v[c] = (row < g.m && (uint32_t)c * 4 < g.k) ? __ldg(src + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        } else if (g.vec2) {  // even k, 8-byte aligned rows: half the load instructions
            const float2* src = reinterpret_cast<const float2*>(g.a + row * g.k);
#pragma unroll
            for (int c = 0; c < KC; ++c) {
                const uint32_t kk = (uint32_t)c * 4;
                const float2 lo2 = (row < g.m && kk < g.k) ? __ldg(src + 2 * c) : make_float2(0.f, 0.f);
                const float2 hi2 = (row < g.m && kk + 2 < g.k) ? __ldg(src + 2 * c + 1) : make_float2(0.f, 0.f);
                v[c] = make_float4(lo2.x, lo2.y, hi2.x, hi2.y);
            }
        } else {
            const float* src = g.a + row * g.k;
#pragma unroll
            for (int c = 0; c < KC; ++c) {
                float e[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t kk = (uint32_t)c * 4 + q;
                    e[q] = (row < g.m && kk < g.k) ? __ldg(src + kk) : 0.f;
                }
                v[c] = make_float4(e[0], e[1], e[2], e[3]);
            }
        }
    };

    constexpr uint32_t IDESC = idesc_tf32<NP>();
    uint32_t parity = 0;
    uint32_t tile = blockIdx.x;
    if (tile < g.tiles) load(tile);
    for (; tile < g.tiles; tile += gridDim.x) {
        // the previous tile's MMAs completed (mbarrier) before its epilogue: smem is free
#pragma unroll
        for (int c = 0; c < KC; ++c) {
            float4 hi, lo;
            hi.x = rna_tf32(v[c].x), lo.x = rna_tf32(v[c].x - hi.x);
            hi.y = rna_tf32(v[c].y), lo.y = rna_tf32(v[c].y - hi.y);
            hi.z = rna_tf32(v[c].z), lo.z = rna_tf32(v[c].z - hi.z);
            hi.w = rna_tf32(v[c].w), lo.w = rna_tf32(v[c].w - hi.w);
            *reinterpret_cast<float4*>(s_ahi + c * A_CH + t * 16) = hi;
            *reinterpret_cast<float4*>(s_alo + c * A_CH + t * 16) = lo;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy stores -> tensor core
        __syncthreads();
        if (t == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t ahi = smem_u32(s_ahi), alo = smem_u32(s_alo);
            const uint32_t whi = smem_u32(s_whi), wlo = smem_u32(s_wlo);
#pragma unroll
            for (int s = 0; s < KP / 8; ++s) {
                const uint64_t dahi = smem_desc(ahi + 2 * s * A_CH, A_CH, 128);
                const uint64_t dalo = smem_desc(alo + 2 * s * A_CH, A_CH, 128);
                const uint64_t dwhi = smem_desc(whi + 2 * s * W_CH, W_CH, 128);
                const uint64_t dwlo = smem_desc(wlo + 2 * s * W_CH, W_CH, 128);
                mma_tf32(tmem, dalo, dwhi, IDESC, s > 0 ? 1u : 0u);  // small terms first
                mma_tf32(tmem, dahi, dwlo, IDESC, 1u);
                mma_tf32(tmem, dahi, dwhi, IDESC, 1u);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar_a)
                         : "memory");
        }
        const uint32_t next = tile + gridDim.x;
        if (next < g.tiles) load(next);  // in flight during the MMAs and the epilogue
        mbar_wait(bar_a, parity);
        parity ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;");
        float acc[NP];
#pragma unroll
        for (int c = 0; c < NP; c += 16) tmem_ld16(tmem + ((warp * 32u) << 16) + (uint32_t)c, acc + c);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");

        const uint64_t row = (uint64_t)tile * TM + warp * 32 + lane;
        if (row < g.m) {
            if (g.epilogue == 1) {
#pragma unroll
                for (int j = 0; j < NP; ++j) {
                    const float x = acc[j] + ((uint32_t)j < nj ? __ldg(g.bias + j0 + j) : 0.f);
                    acc[j] = x > 0.f ? x : 0.f;
                }
            } else if (g.epilogue == 2) {
                const float sc = (float)g.row_scale[row];
#pragma unroll
                for (int j = 0; j < NP; ++j) acc[j] *= sc;
            }
            float* o = g.out + row * g.n + j0;
            if (nj == (uint32_t)NP && g.n % 4 == 0 && ((uintptr_t)o % 16 == 0)) {
#pragma unroll
                for (int j = 0; j < NP; j += 4)
                    *reinterpret_cast<float4*>(o + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < NP; ++j)
                    if ((uint32_t)j < nj) o[j] = acc[j];
            }
        }
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
}

// ---------------------------------------------------------------------------
// TMA-fed variant (k % 4 == 0, 16-byte aligned A): the A tile arrives by
// cp.async.bulk.tensor (box 32 fp32 x 128 rows per K slice, SWIZZLE_128B),
// which IS the canonical SW128 K-major operand layout, so the raw fp32 tile
// is A_hi as the tensor core reads it (tf32 = the top 19 bits).  The only
// register pass is lo = x - trunc_tf32(x) (lo_part2) written elementwise at the
// same offsets (linear, conflict-free).  An S-deep ring of stages keeps S
// tiles of HBM reads in flight while the CTA converts, multiplies and writes.
// Two MMAs per K step: A_hi x [W_hi ; W_lo] (N = 2*NP, TMEM columns
// [0,NP) and [NP,2NP)) and A_lo x W_hi (N = NP, onto columns [0,NP)); the
// epilogue adds the two column halves.
// ---------------------------------------------------------------------------

// UMMA descriptor, SWIZZLE_128B K-major: rows of 128 B, 8-row atoms at SBO =
// 1024 B (LBO unused, 1), layout type 2.  Atoms must be 1024-byte aligned.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
           (2ull << 61);
}

template <int KP, int NP>
struct TmaCfg {
    static constexpr int SL = KP / 32;           // K slices (128-byte rows)
    static constexpr uint32_t SLICE = TM * 128;  // one slice of a 128-row tile (16 KB)
    static constexpr uint32_t STAGE = SL * SLICE;
    static constexpr uint32_t WSL = 2 * NP * 128;  // one slice of [W_hi^T ; W_lo^T]
    static constexpr uint32_t WB = SL * WSL;
    static constexpr uint32_t BUDGET = 224 * 1024;
    static constexpr uint32_t OSTRIDE = NP + 1;              // output staging row stride (floats)
    static constexpr uint32_t OUTB = 8 * 32 * OSTRIDE * 4;   // per-warp 32-row output staging
    static constexpr int S0 = (int)((BUDGET - WB - OUTB) / STAGE);
    static constexpr int S = S0 > 4 ? 4 : S0;  // TMA stages in flight
    static constexpr size_t SMEM = (size_t)S * STAGE + WB + OUTB + 1024;  // + alignment slack
    // TMEM columns: two accumulators [hi | lo-correction] of 2*NP, then two
    // A_lo tiles of KP (lane = row, one tf32 per column)
    static constexpr uint32_t ACC = 2 * NP;
    static constexpr uint32_t LO0 = 2 * ACC;
    static constexpr uint32_t NEED = LO0 + 2 * KP;
    static constexpr uint32_t TCOLS = NEED <= 32 ? 32 : NEED <= 64 ? 64 : NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
    static_assert(NEED <= 512, "TMEM");
    // AT: the converters also store A_hi (the raw tile) into TMEM and both MMAs
    // are TS, so the tensor core reads only W from shared memory
    static constexpr bool AT_FITS = LO0 + 4 * KP <= 512;
    static constexpr uint32_t TCOLS_AT = AT_FITS ? (LO0 + 4 * KP <= 256 ? 256 : 512) : 512;
};

__device__ __forceinline__ float trunc_tf32(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__device__ __forceinline__ float lo_part(float x) { return rna_tf32(x - trunc_tf32(x)); }

// The converters' split of a streamed operand: the MMA reads an fp32 operand
// as tf32 by dropping its low 13 bits, so the raw x serves as hi, and
// lo = x - trunc(x) (exact in fp32) as the correction, which the MMA
// truncates in turn: error <= 2^-20 |x| per operand, against 2^-21 when lo is
// rounded to nearest first (GNNA_TF32_LO_RNA=1, three more instructions per
// element).  Two elements per packed FADD2.
#ifndef GNNA_TF32_LO_RNA
#define GNNA_TF32_LO_RNA 0
#endif
__device__ __forceinline__ float2 lo_part2(float a, float b) {
#if GNNA_TF32_LO_RNA
    return make_float2(lo_part(a), lo_part(b));
#else
    return __fadd2_rn(make_float2(a, b), make_float2(-trunc_tf32(a), -trunc_tf32(b)));
#endif
}

// 16 registers -> 16 consecutive TMEM columns of this warp's 32 lanes.
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
            taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
        "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
        "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
        "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
        "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])));
}

// A from TMEM (A_lo), B from shared memory.
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t db, uint32_t idesc,
                                            uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(db), "r"(idesc), "r"(acc));
}

// Warp roles: two groups of four warps (group b = warps 4b..4b+3, thread =
// TMEM lane = tile row) take alternate tiles (b = tile index & 1): each
// converts A_lo into its TMEM buffer and runs the epilogue of its tile, so
// one group's epilogue overlaps the other's conversion.  Warp 8 issues the
// TMA loads and the MMAs.  Hand-offs are mbarriers: full[s] (TMA ->
// converters), lo_full[b] (128 arrivals of group b -> MMA warp), mma_bar[b]
// (tcgen05.commit -> group b's epilogue and the stage refill).
constexpr int TC_CONV = 2 * TM;
constexpr int TC_THREADS = TC_CONV + 32;

template <int KP, int NP, bool AT>
__global__ void __launch_bounds__(TC_THREADS, 1) k6_gemm_tc_tma(const __grid_constant__ CUtensorMap tmap, TcArgs g) {
    using C = TmaCfg<KP, NP>;
    constexpr int S = C::S;
    static_assert(KP % 32 == 0 && S >= 2 && (!AT || C::AT_FITS), "config");
    constexpr uint32_t TCOLS = AT ? C::TCOLS_AT : C::TCOLS;
    constexpr uint32_t LOB_COLS = AT ? 2 * KP : KP;  // per buffer: A_lo [| A_hi]
    extern __shared__ unsigned char smem_raw[];
    __shared__ uint64_t full[S];
    __shared__ uint64_t lo_full[2];
    __shared__ uint64_t mma_bar[2];
    __shared__ uint32_t tmem_slot;
    const uint32_t raw_a = smem_u32(smem_raw);
    const uint32_t base = (raw_a + 1023u) & ~1023u;
    unsigned char* base_p = smem_raw + (base - raw_a);
    const uint32_t w_a = base + S * C::STAGE;
    unsigned char* w_p = base_p + S * C::STAGE;
    float* ostage = reinterpret_cast<float*>(w_p + C::WB);

    const uint32_t t = threadIdx.x, warp = t / 32, lane = t % 32;
    const uint32_t j0 = blockIdx.y * NP;
    const uint32_t nj = g.n - j0 < (uint32_t)NP ? g.n - j0 : (uint32_t)NP;
    const uint32_t my_tiles = g.tiles > blockIdx.x ? (g.tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

    auto issue = [&](uint32_t i) {  // one thread: TMA of this CTA's i-th tile into stage i % S
        const uint32_t s = i % S, tile = blockIdx.x + i * gridDim.x;
        const uint32_t bar = smem_u32(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(C::STAGE) : "memory");
#pragma unroll
        for (int sl = 0; sl < C::SL; ++sl)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                "[%4];" ::"r"(base + s * C::STAGE + sl * C::SLICE),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(sl * 32), "r"(tile * TM), "r"(bar)
                : "memory");
    };

    if (t == TC_CONV) {  // MMA warp, lane 0: barriers, then the first S loads (overlap the W staging below)
        for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
        for (int b = 0; b < 2; ++b) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&lo_full[b])), "r"(TM));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mma_bar[b])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
        for (uint32_t i = 0; i < (uint32_t)S && i < my_tiles; ++i) issue(i);
    }
    if (t < TC_CONV) {
        // [W_hi^T ; W_lo^T]: 2*NP rows, K-major, 128-byte swizzle (chunk ^= row % 8);
        // all loads first so their latencies overlap
        constexpr int PER = NP * KP / TC_CONV;
        float wv[PER];
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const uint32_t e = t + q * TC_CONV, nn = e / KP, kk = e % KP;
            wv[q] = (nn < nj && kk < g.k) ? __ldg(g.w + (uint64_t)kk * g.n + j0 + nn) : 0.f;
        }
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const uint32_t e = t + q * TC_CONV, nn = e / KP, kk = e % KP;
            const float hi = rna_tf32(wv[q]), lo = rna_tf32(wv[q] - hi);
            const uint32_t sl = kk / 32, c = (kk % 32) / 4, b = (kk % 4) * 4;
            const uint32_t r0 = nn, r1 = NP + nn;
            *reinterpret_cast<float*>(w_p + sl * C::WSL + (r0 / 8) * 1024 + (r0 % 8) * 128 + ((c ^ (r0 % 8)) * 16) +
                                      b) = hi;
            *reinterpret_cast<float*>(w_p + sl * C::WSL + (r1 / 8) * 1024 + (r1 % 8) * 128 + ((c ^ (r1 % 8)) * 16) +
                                      b) = lo;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // W (generic stores) -> tensor core
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                     "r"(TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_slot;

    if (warp == 8) {
        // MMA issuer + stage refills
        constexpr uint32_t IDESC_2N = idesc_tf32<2 * NP>();
        constexpr uint32_t IDESC_N = idesc_tf32<NP>();
        for (uint32_t i = 0; i < my_tiles; ++i) {
            const uint32_t s = i % S, b = i & 1u;
            mbar_wait(smem_u32(&lo_full[b]), (i >> 1) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (lane == 0) {
                const uint32_t a_hi = base + s * C::STAGE;
                const uint32_t d = tmem + b * C::ACC, a_lo = tmem + C::LO0 + b * LOB_COLS;
#pragma unroll
                for (int sl = 0; sl < C::SL; ++sl)
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t ao = sl * C::SLICE + q * 32, bo = sl * C::WSL + q * 32;
                        if (AT)
                            mma_tf32_ts(d, a_lo + KP + sl * 32 + q * 8, smem_desc_sw128(w_a + bo), IDESC_2N,
                                        (sl | q) ? 1u : 0u);
                        else
                            mma_tf32(d, smem_desc_sw128(a_hi + ao), smem_desc_sw128(w_a + bo), IDESC_2N,
                                     (sl | q) ? 1u : 0u);
                        mma_tf32_ts(d, a_lo + sl * 32 + q * 8, smem_desc_sw128(w_a + bo), IDESC_N, 1u);
                    }
                asm volatile(
                    "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                        smem_u32(&mma_bar[b]))
                    : "memory");
            }
            __syncwarp();
            if (i >= 1) {
                const uint32_t j = i - 1;
                mbar_wait(smem_u32(&mma_bar[j & 1u]), (j >> 1) & 1u);  // MMA(j) has read stage j % S
                if (lane == 0 && j + S < my_tiles) issue(j + S);
                __syncwarp();
            }
        }
    } else {
        // converters / epilogue: thread r = TMEM lane r = tile row r
        const uint32_t grp = warp / 4, wq = warp % 4;
        const uint32_t lane_off = (wq * 32u) << 16;
        const uint32_t r = wq * 32 + lane, r8 = r % 8;
        const uint32_t row_off = (r / 8) * 1024 + r8 * 128;  // this thread's row inside a slice
        for (uint32_t i = grp; i < my_tiles; i += 2) {
            {
                const uint32_t s = i % S, b = i & 1u;
                mbar_wait(smem_u32(&full[s]), (i / S) & 1u);
                // lo = x - trunc_tf32(x) of this thread's row (lo_part2), read from the
                // swizzled tile (8 consecutive lanes hit 8 distinct bank groups)
                const unsigned char* stg = base_p + s * C::STAGE + row_off;
#pragma unroll
                for (int sl = 0; sl < C::SL; ++sl) {
                    float4 x[8];
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        x[c] = *reinterpret_cast<const float4*>(stg + sl * C::SLICE + ((c ^ r8) * 16));
                    float lo[32];
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float2 l01 = lo_part2(x[c].x, x[c].y), l23 = lo_part2(x[c].z, x[c].w);
                        lo[4 * c] = l01.x, lo[4 * c + 1] = l01.y, lo[4 * c + 2] = l23.x, lo[4 * c + 3] = l23.y;
                    }
                    const uint32_t col = tmem + lane_off + C::LO0 + b * LOB_COLS + sl * 32;
                    tmem_st16(col, lo);
                    tmem_st16(col + 16, lo + 16);
                    if (AT) {
                        tmem_st16(col + KP, reinterpret_cast<const float*>(x));
                        tmem_st16(col + KP + 16, reinterpret_cast<const float*>(x) + 16);
                    }
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;");
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&lo_full[b])) : "memory");
            }
            const uint32_t j = i, bj = j & 1u;
            mbar_wait(smem_u32(&mma_bar[bj]), (j >> 1) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;");
            float acc[2 * NP];
#pragma unroll
            for (int c = 0; c < 2 * NP; c += 16) tmem_ld16(tmem + lane_off + bj * C::ACC + (uint32_t)c, acc + c);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;");  // ordered before the next lo_full arrival
#pragma unroll
            for (int q = 0; q < NP; ++q) acc[q] += acc[NP + q];

            const uint64_t row0 = (uint64_t)(blockIdx.x + j * gridDim.x) * TM + wq * 32;
            const uint64_t row = row0 + lane;
            if (row < g.m) {
                if (g.epilogue == 1) {
#pragma unroll
                    for (int q = 0; q < NP; ++q) {
                        const float x = acc[q] + ((uint32_t)q < nj ? __ldg(g.bias + j0 + q) : 0.f);
                        acc[q] = x > 0.f ? x : 0.f;
                    }
                } else if (g.epilogue == 2) {
                    const float sc = (float)g.row_scale[row];
#pragma unroll
                    for (int q = 0; q < NP; ++q) acc[q] *= sc;
                }
            }
            if (gridDim.y == 1) {
                // the warp's 32 output rows are one contiguous run of 32*n floats:
                // stage them (row stride NP+1: conflict-free) and store coalesced
                float* st = ostage + warp * 32 * C::OSTRIDE;
#pragma unroll
                for (int q = 0; q < NP; ++q) st[lane * C::OSTRIDE + q] = acc[q];
                __syncwarp();
                const uint32_t rows = row0 >= g.m ? 0u : (g.m - row0 < 32u ? (uint32_t)(g.m - row0) : 32u);
                const uint32_t total = rows * g.n;
                float* o = g.out + row0 * g.n;
                uint32_t rr = lane / g.n, cc = lane % g.n;
                const uint32_t dr = 32u / g.n, dc = 32u % g.n;
                for (uint32_t e = lane; e < total; e += 32) {
                    o[e] = st[rr * C::OSTRIDE + cc];
                    rr += dr, cc += dc;
                    if (cc >= g.n) cc -= g.n, ++rr;
                }
                __syncwarp();
            } else if (row < g.m) {
                float* o = g.out + row * g.n + j0;
                if (nj == (uint32_t)NP && g.n % 4 == 0 && ((uintptr_t)o % 16 == 0)) {
#pragma unroll
                    for (int q = 0; q < NP; q += 4)
                        *reinterpret_cast<float4*>(o + q) = make_float4(acc[q], acc[q + 1], acc[q + 2], acc[q + 3]);
                } else {
#pragma unroll
                    for (int q = 0; q < NP; ++q)
                        if ((uint32_t)q < nj) o[q] = acc[q];
                }
            }
        }
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
}

// The same product with the roles split (K 128 or N blocks of 64; GNNA_TC_SPLIT=0/1 forces): warps
// 0-3 only convert (A_lo into a LOB-deep TMEM ring), warps 4-11 only run the
// epilogue (two groups, one per TMEM accumulator, alternate tiles), warp 12
// issues the MMAs, warp 13 refills the TMA ring as each stage's MMAs commit.  In the two-group kernel above a
// group converts tile i + 2 only after its epilogue of tile i, so the tensor
// pipe waited on epilogue + conversion every tile; here conversion runs up to
// LOB tiles ahead and the epilogue trails.  It wins where conversion or the
// epilogue is heavy (K 128, 64 output columns); on the narrow C3 products the
// two-group kernel stays ahead, and every tile's MMAs are bound by shared-memory reads
// (tensor-core A reads + TMA writes + converter loads, ~128 B/cycle; a clock64
// trace showed 24 MMAs taking ~1,600 cycles per 128-row tile at C3).
constexpr int TCS_THREADS = 3 * TM + 64;

template <int KP, int NP>
struct TcSplitCfg {
    using C = TmaCfg<KP, NP>;
    static constexpr uint32_t ACC = C::ACC;
    static constexpr int LOB = 2 * ACC + 3 * KP <= 512 ? 3 : 2;
    static constexpr uint32_t LO0 = 2 * ACC;
    static constexpr uint32_t NEED = LO0 + LOB * KP;
    static constexpr uint32_t TCOLS = NEED <= 32 ? 32 : NEED <= 64 ? 64 : NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
    static_assert(NEED <= 512, "TMEM");
};

template <int KP, int NP>
__global__ void __launch_bounds__(TCS_THREADS, 1)
    k6_gemm_tc_tma_split(const __grid_constant__ CUtensorMap tmap, TcArgs g) {
    using C = TmaCfg<KP, NP>;
    using D = TcSplitCfg<KP, NP>;
    constexpr int S = C::S, LOB = D::LOB;
    static_assert(KP % 32 == 0 && S >= 2, "config");
    extern __shared__ unsigned char smem_raw[];
    __shared__ uint64_t full[S], empty[S], lo_full[LOB], lo_free[LOB], acc_full[2], acc_free[2];
    __shared__ uint32_t tmem_slot;
    const uint32_t raw_a = smem_u32(smem_raw);
    const uint32_t base = (raw_a + 1023u) & ~1023u;
    unsigned char* base_p = smem_raw + (base - raw_a);
    const uint32_t w_a = base + S * C::STAGE;
    unsigned char* w_p = base_p + S * C::STAGE;
    float* ostage = reinterpret_cast<float*>(w_p + C::WB);

    const uint32_t t = threadIdx.x, warp = t / 32, lane = t % 32;
    const uint32_t j0 = blockIdx.y * NP;
    const uint32_t nj = g.n - j0 < (uint32_t)NP ? g.n - j0 : (uint32_t)NP;
    const uint32_t my_tiles = g.tiles > blockIdx.x ? (g.tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

    auto issue = [&](uint32_t i) {  // one thread: TMA of this CTA's i-th tile into stage i % S
        const uint32_t s = i % S, tile = blockIdx.x + i * gridDim.x;
        const uint32_t bar = smem_u32(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(C::STAGE) : "memory");
#pragma unroll
        for (int sl = 0; sl < C::SL; ++sl)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                "[%4];" ::"r"(base + s * C::STAGE + sl * C::SLICE),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(sl * 32), "r"(tile * TM), "r"(bar)
                : "memory");
    };

    if (t == 3 * TM) {  // MMA warp, lane 0: barriers, then the first S loads (overlap the W staging below)
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])));
        }
        for (int b = 0; b < LOB; ++b) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&lo_full[b])), "r"(TM));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&lo_free[b])));
        }
        for (int a = 0; a < 2; ++a) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&acc_full[a])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&acc_free[a])), "r"(TM));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
        for (uint32_t i = 0; i < (uint32_t)S && i < my_tiles; ++i) issue(i);
    }
    if (t < 2 * TM) {
        // [W_hi^T ; W_lo^T]: 2*NP rows, K-major, 128-byte swizzle (chunk ^= row % 8)
        constexpr int PER = NP * KP / (2 * TM);
        float wv[PER];
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const uint32_t e = t + q * 2 * TM, nn = e / KP, kk = e % KP;
            wv[q] = (nn < nj && kk < g.k) ? __ldg(g.w + (uint64_t)kk * g.n + j0 + nn) : 0.f;
        }
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const uint32_t e = t + q * 2 * TM, nn = e / KP, kk = e % KP;
            const float hi = rna_tf32(wv[q]), lo = rna_tf32(wv[q] - hi);
            const uint32_t sl = kk / 32, c = (kk % 32) / 4, b = (kk % 4) * 4;
            const uint32_t r0 = nn, r1 = NP + nn;
            *reinterpret_cast<float*>(w_p + sl * C::WSL + (r0 / 8) * 1024 + (r0 % 8) * 128 + ((c ^ (r0 % 8)) * 16) +
                                      b) = hi;
            *reinterpret_cast<float*>(w_p + sl * C::WSL + (r1 / 8) * 1024 + (r1 % 8) * 128 + ((c ^ (r1 % 8)) * 16) +
                                      b) = lo;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // W (generic stores) -> tensor core
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                     "r"(D::TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_slot;

    if (warp == 12) {
        constexpr uint32_t IDESC_2N = idesc_tf32<2 * NP>();
        constexpr uint32_t IDESC_N = idesc_tf32<NP>();
        for (uint32_t i = 0; i < my_tiles; ++i) {
            const uint32_t s = i % S, b = i % LOB, a = i & 1u;
            mbar_wait(smem_u32(&lo_full[b]), (i / LOB) & 1u);        // converters done (stage s has landed)
            if (i >= 2) mbar_wait(smem_u32(&acc_free[a]), ((i - 2) >> 1) & 1u);  // epilogue read tile i - 2
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (lane == 0) {
                const uint32_t a_hi = base + s * C::STAGE;
                const uint32_t d = tmem + a * D::ACC, a_lo = tmem + D::LO0 + b * KP;
#pragma unroll
                for (int sl = 0; sl < C::SL; ++sl)
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t ao = sl * C::SLICE + q * 32, bo = sl * C::WSL + q * 32;
                        mma_tf32(d, smem_desc_sw128(a_hi + ao), smem_desc_sw128(w_a + bo), IDESC_2N,
                                 (sl | q) ? 1u : 0u);
                        mma_tf32_ts(d, a_lo + sl * 32 + q * 8, smem_desc_sw128(w_a + bo), IDESC_N, 1u);
                    }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(&acc_full[a]))
                             : "memory");
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(&lo_free[b]))
                             : "memory");
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(&empty[s]))
                             : "memory");
            }
            __syncwarp();
        }
    } else if (warp == 13) {
        if (lane == 0)
            for (uint32_t i = S; i < my_tiles; ++i) {
                mbar_wait(smem_u32(&empty[(i - S) % S]), ((i - S) / S) & 1u);
                issue(i);
            }
    } else if (warp < 4) {
        // converters: thread r = TMEM lane r = tile row r
        const uint32_t lane_off = (warp * 32u) << 16;
        const uint32_t r = warp * 32 + lane, r8 = r % 8;
        const uint32_t row_off = (r / 8) * 1024 + r8 * 128;
        for (uint32_t i = 0; i < my_tiles; ++i) {
            const uint32_t s = i % S, b = i % LOB;
            mbar_wait(smem_u32(&full[s]), (i / S) & 1u);
            if (i >= (uint32_t)LOB) mbar_wait(smem_u32(&lo_free[b]), ((i - LOB) / LOB) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const unsigned char* stg = base_p + s * C::STAGE + row_off;
#pragma unroll
            for (int sl = 0; sl < C::SL; ++sl) {
                float4 x[8];
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    x[c] = *reinterpret_cast<const float4*>(stg + sl * C::SLICE + ((c ^ r8) * 16));
                float lo[32];
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float2 l01 = lo_part2(x[c].x, x[c].y), l23 = lo_part2(x[c].z, x[c].w);
                    lo[4 * c] = l01.x, lo[4 * c + 1] = l01.y, lo[4 * c + 2] = l23.x, lo[4 * c + 3] = l23.y;
                }
                const uint32_t col = tmem + lane_off + D::LO0 + b * KP + sl * 32;
                tmem_st16(col, lo);
                tmem_st16(col + 16, lo + 16);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;");
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&lo_full[b])) : "memory");
        }
    } else {
        // epilogue: warps 4-7 take the even tiles (accumulator 0), warps 8-11
        // the odd ones (accumulator 1); thread = TMEM lane (warp % 4) * 32 + lane = tile row
        const uint32_t grp = (warp - 4) / 4, wq = warp % 4;
        const uint32_t lane_off = (wq * 32u) << 16;
        for (uint32_t i = grp; i < my_tiles; i += 2) {
            const uint32_t a = i & 1u;
            mbar_wait(smem_u32(&acc_full[a]), (i >> 1) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;");
            float acc[2 * NP];
#pragma unroll
            for (int c = 0; c < 2 * NP; c += 16) tmem_ld16(tmem + lane_off + a * D::ACC + (uint32_t)c, acc + c);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;");
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&acc_free[a])) : "memory");
#pragma unroll
            for (int q = 0; q < NP; ++q) acc[q] += acc[NP + q];
            const uint64_t row0 = (uint64_t)(blockIdx.x + i * gridDim.x) * TM + wq * 32;
            const uint64_t row = row0 + lane;
            if (row < g.m) {
                if (g.epilogue == 1) {
#pragma unroll
                    for (int q = 0; q < NP; ++q) {
                        const float x = acc[q] + ((uint32_t)q < nj ? __ldg(g.bias + j0 + q) : 0.f);
                        acc[q] = x > 0.f ? x : 0.f;
                    }
                } else if (g.epilogue == 2) {
                    const float sc = (float)g.row_scale[row];
#pragma unroll
                    for (int q = 0; q < NP; ++q) acc[q] *= sc;
                }
            }
            if (gridDim.y == 1) {
                float* st = ostage + (warp - 4) * 32 * C::OSTRIDE;
#pragma unroll
                for (int q = 0; q < NP; ++q) st[lane * C::OSTRIDE + q] = acc[q];
                __syncwarp();
                const uint32_t rows = row0 >= g.m ? 0u : (g.m - row0 < 32u ? (uint32_t)(g.m - row0) : 32u);
                const uint32_t total = rows * g.n;
                float* o = g.out + row0 * g.n;
                uint32_t rr = lane / g.n, cc = lane % g.n;
                const uint32_t dr = 32u / g.n, dc = 32u % g.n;
                for (uint32_t e = lane; e < total; e += 32) {
                    o[e] = st[rr * C::OSTRIDE + cc];
                    rr += dr, cc += dc;
                    if (cc >= g.n) cc -= g.n, ++rr;
                }
                __syncwarp();
            } else if (row < g.m) {
                float* o = g.out + row * g.n + j0;
                if (nj == (uint32_t)NP && g.n % 4 == 0 && ((uintptr_t)o % 16 == 0)) {
#pragma unroll
                    for (int q = 0; q < NP; q += 4)
                        *reinterpret_cast<float4*>(o + q) = make_float4(acc[q], acc[q + 1], acc[q + 2], acc[q + 3]);
                } else {
#pragma unroll
                    for (int q = 0; q < NP; ++q)
                        if ((uint32_t)q < nj) o[q] = acc[q];
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(D::TCOLS));
}

// cudaFuncSetAttribute is per device: each kernel instance remembers the
// devices it was configured on (one bit per device ordinal).
template <class K>
void smem_attr_once(std::atomic<uint64_t>& done, K kern, int device, size_t bytes) {
    const uint64_t bit = 1ull << (device & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    GNNA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    done.fetch_or(bit, std::memory_order_release);
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

template <int KP, int NP>
bool launch_tc_tma(gnna_ctx* ctx, const TcArgs& g) {
    auto encode = tensor_map_encoder();
    if (!encode) return false;
    CUtensorMap map;
    const cuuint64_t dims[2] = {g.k, g.m};
    const cuuint64_t strides[1] = {(cuuint64_t)g.k * 4};
    const cuuint32_t box[2] = {32, (cuuint32_t)TM};
    const cuuint32_t es[2] = {1, 1};
    if (encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(g.a), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    using C = TmaCfg<KP, NP>;
    // split roles for K 128 or 64-column blocks (410k x 128 -> 64: 141 -> 94 us,
    // 1M x 64 -> 64: 93.5 -> 87); the two-group kernel for the narrow C3
    // products (96 -> 16: 33.3 vs 37.0 us, 16 -> 22: 21.6 vs 22.3)
    static const int split_env = [] {
        const char* e = std::getenv("GNNA_TC_SPLIT");  // A/B switch: 0 / 1 force either kernel
        return e && *e ? std::atoi(e) : -1;
    }();
    const bool split = split_env >= 0 ? split_env != 0 : (KP >= 128 || NP >= 64);
    static const bool at_on = [] {
        const char* e = std::getenv("GNNA_TC_AT");  // A/B switch (0: A_hi read from shared memory)
        return !(e && *e == '0');
    }();
    auto kern = split ? k6_gemm_tc_tma_split<KP, NP>
                      : (C::AT_FITS && at_on) ? k6_gemm_tc_tma<KP, NP, C::AT_FITS> : k6_gemm_tc_tma<KP, NP, false>;
    static std::atomic<uint64_t> attr{0};
    smem_attr_once(attr, kern, ctx->device, C::SMEM);
    const uint32_t cols = (g.n + NP - 1) / NP;
    const uint32_t slots = (uint32_t)ctx->num_sms / cols;
    dim3 grid(g.tiles < slots ? g.tiles : (slots ? slots : 1), cols);
    kern<<<grid, split ? TCS_THREADS : TC_THREADS, C::SMEM, ctx->stream>>>(map, g);
    launched(ctx, "k6_gemm_tc_tma");
    return true;
}

template <int KP>
bool launch_tma_n(gnna_ctx* ctx, const TcArgs& g) {
    if (g.n <= 16) return launch_tc_tma<KP, 16>(ctx, g);
    if (g.n <= 32 || KP > 96) return launch_tc_tma<KP, 32>(ctx, g);  // KP 128: 32-column blocks keep 2 stages
    if constexpr (KP <= 96) return launch_tc_tma<KP, 64>(ctx, g);
    return false;
}

template <int KP, int NP>
void launch_tc(gnna_ctx* ctx, const TcArgs& g0) {
    TcArgs g = g0;
    constexpr size_t smem = (size_t)2 * (KP / 4) * TM * 16 + (size_t)2 * (KP / 4) * NP * 16;
    auto kern = k6_gemm_tc<KP, NP>;
    static std::atomic<uint64_t> attr{0};
    smem_attr_once(attr, kern, ctx->device, smem);
    static int per_sm = [&] {
        int b = 0;
        GNNA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, TM, smem));
        return b < 1 ? 1 : b;
    }();
    const uint32_t cols = (g.n + NP - 1) / NP;
    const uint32_t slots = (uint32_t)(ctx->num_sms * per_sm) / cols;
    dim3 grid(g.tiles < slots ? g.tiles : (slots ? slots : 1), cols);
    kern<<<grid, TM, smem, ctx->stream>>>(g);
    GNNA_CUDA(cudaGetLastError());
    launched(ctx, "k6_gemm_tc");
}

template <int KP>
void launch_tc_n(gnna_ctx* ctx, const TcArgs& g) {
    if (g.n <= 16)
        launch_tc<KP, 16>(ctx, g);
    else if (g.n <= 32)
        launch_tc<KP, 32>(ctx, g);
    else
        launch_tc<KP, 64>(ctx, g);
}

// ---------------------------------------------------------------------------
// dW = A^T B on tcgen05 (the backward of the update GEMM, gcn/gin_layer_backward):
// a reduction over all m rows.  A (m x p) and B (m x q) are row-major, so as
// MMA operands (M = feature of A, N = feature of B, K = row) both are
// MN-major.  For tf32 the MN-major smem layout is the 128-byte swizzle with
// 32-byte atomicity (layout type 1): 32-feature slices of BK rows, 4-row
// 512-byte K atoms; the TMA mode CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B writes
// exactly that, so the raw TMA'd stage IS A_hi / B_hi.
//   * stage (S-deep ring): A[PS slices] | B_hi[QS] | B_lo[QS], where B_lo =
//     x - trunc(x) (lo_part2) is written elementwise by the converter warps at
//     the same swizzled offsets, one LBO after B_hi: [B_hi | B_lo] is ONE
//     N = 64*QS operand;
//   * A_lo goes to TMEM (K-major there: lane = feature, column = row),
//     written by the converter thread that owns the feature lane;
//   * per K step: A_hi x [B_hi | B_lo] (SS, columns [0,32QS) and
//     [32QS,64QS)) + A_lo x B_hi (TS, onto [0,32QS)), accumulated in TMEM
//     for the CTA's whole run of BK-row blocks (split-K); the epilogue adds
//     the two column halves (packed QS = 0 below: both MMAs are N = 32 over
//     the one [B_hi | B_lo] slice, so A_lo x B_lo lands in columns 16-31 too);
//   * warp 4 issues the MMAs, warp 5 (PROD) refills each stage as its MMAs
//     commit, warps 0-3 convert.
// M = 128 reads 4 A slices from the stage base: the 4 - PS phantom slices
// alias the following bytes (in bounds) and only feed discarded rows of D.
// Per-CTA partials are summed by k_reduce_partials in a fixed slice order
// (deterministic; GNNA_TN_SEQ_REDUCE=1 keeps the sequential CTA-order k6_tn_reduce).
// ---------------------------------------------------------------------------
// QS = 0 is the packed form for q <= 16: ONE B slice holds [B_hi | B_lo]
// (the TMA writes B into columns 0-15, the columns past q arrive zero-filled,
// and the converters write B_lo into columns 16-31 of the same swizzled
// rows), so the SS MMA is N = 32 and the stage has no separate B_lo slice.
// BK = rows per block (one TMA box per 32-feature slice): 128 where three
// such stages fit, else 64.  Each tcgen05.mma here is M 128 x N 32..64 x K 8,
// which costs a fixed ~45 cycles (scripts/micro/mma_rate.cu), so a block's
// MMA time is its instruction count; bigger blocks halve the per-block
// handoffs and commits (C3 dW1: 43.4 -> 39.0 us).
template <int PS, int QS, int BK>
struct TnCfg {
    static constexpr uint32_t SL = BK * 128;  // one 32-feature slice of a block (8 / 16 KB)
    static constexpr uint32_t QB = QS ? QS : 1;  // B slices the TMA loads
    static constexpr uint32_t AH = 0, BH = PS * SL, BL = BH + QB * SL;
    static constexpr uint32_t STAGE = (PS + QB + QS) * SL;
    static constexpr uint32_t TAIL = (4 - PS) * SL;  // phantom A slices past the last stage
    static constexpr int S0 = (int)((224u * 1024u - TAIL) / STAGE);
    static constexpr int S = S0 > 8 ? 8 : S0;
    static constexpr size_t SMEM = (size_t)S * STAGE + TAIL + 1024;
    static constexpr uint32_t ND = QS ? 64 * QS : 32;        // accumulator columns [hi.hi | hi.lo]
    static constexpr int LOB = BK >= 128 ? 3 : 4;           // A_lo ring depth (TMEM)
    static constexpr uint32_t LO0 = ND;                     // A_lo buffers: LOB x BK columns
    static constexpr uint32_t NEED = LO0 + LOB * BK;
    static constexpr uint32_t TCOLS = NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
    static_assert(NEED <= 512, "TMEM");
};

// tf32, D f32, M = 128; A and B major-ness as given (bit 15 A, bit 16 B; 1 = MN-major).
template <int N, int AMN, int BMN>
__device__ __forceinline__ constexpr uint32_t idesc_tf32_mj() {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)AMN << 15) | ((uint32_t)BMN << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
}

// MN-major tf32 operand descriptor: layout type 1 (SWIZZLE_128B_BASE32B),
// LBO = stride between 32-element MN groups, SBO = 512 (next 4-row K atom;
// one K=8 MMA spans two).
__device__ __forceinline__ uint64_t smem_desc_mn128(uint32_t addr, uint32_t lbo) {
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)(512 >> 4) << 32) | (1ull << 46) | (1ull << 61);
}

struct TnArgs {
    uint32_t m, p, q;
    uint32_t nblk, bpc;  // BK-row blocks, blocks per CTA
    float* part;         // [gridDim.x][p][q]
};

constexpr int TN_THREADS = TM + 32;

// PROD: a sixth warp refills the ring (waits each stage's `empty` in order
// and re-issues its TMA) instead of the MMA warp between MMAs, so a refill
// never waits for the converters of the next block.
template <int PS, int QS, int BK, bool PROD>
__global__ void __launch_bounds__(TN_THREADS + 32, 1) k6_gemm_tn_tc(const __grid_constant__ CUtensorMap amap,
                                                               const __grid_constant__ CUtensorMap bmap, TnArgs g) {
    using C = TnCfg<PS, QS, BK>;
    constexpr int S = C::S;
    static_assert(S >= 2, "stages");
    extern __shared__ unsigned char smem_raw[];
    constexpr int LOB = C::LOB;
    __shared__ uint64_t full[S], empty[S], ready[LOB], lofree[LOB];
    __shared__ uint32_t tmem_slot;
    const uint32_t raw_a = smem_u32(smem_raw);
    const uint32_t base = (raw_a + 1023u) & ~1023u;
    unsigned char* base_p = smem_raw + (base - raw_a);
    const uint32_t t = threadIdx.x, warp = t / 32, lane = t % 32;
    const uint32_t b0 = blockIdx.x * g.bpc;
    const uint32_t nb = b0 >= g.nblk ? 0u : (g.nblk - b0 < g.bpc ? g.nblk - b0 : g.bpc);
    constexpr uint32_t tx = (PS + C::QB) * C::SL;

    auto issue = [&](uint32_t i) {  // one thread: TMA of local block i into stage i % S
        const uint32_t s = i % S, row = (b0 + i) * BK;
        const uint32_t bar = smem_u32(&full[s]), st = base + s * C::STAGE;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
#pragma unroll
        for (int sl = 0; sl < PS; ++sl)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                "[%4];" ::"r"(st + C::AH + sl * C::SL),
                "l"(reinterpret_cast<uint64_t>(&amap)), "r"(sl * 32), "r"(row), "r"(bar)
                : "memory");
#pragma unroll
        for (int sl = 0; sl < (int)C::QB; ++sl)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                "[%4];" ::"r"(st + C::BH + sl * C::SL),
                "l"(reinterpret_cast<uint64_t>(&bmap)), "r"(sl * 32), "r"(row), "r"(bar)
                : "memory");
    };

    if (t == TM) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])));
        }
        for (int b = 0; b < LOB; ++b) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&ready[b])), "r"(TM));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&lofree[b])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&amap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&bmap)) : "memory");
        for (uint32_t i = 0; i < (uint32_t)S && i < nb; ++i) issue(i);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                     "r"(C::TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_slot;

    if (warp == 4) {
        // packed: A_lo x [B_hi | B_lo] adds the lo x lo term to columns 16-31 as well
        constexpr uint32_t ID_SS = idesc_tf32_mj<C::ND, 1, 1>();
        constexpr uint32_t ID_TS = idesc_tf32_mj<QS ? 32 * QS : 32, 0, 1>();
        for (uint32_t i = 0; i < nb; ++i) {
            const uint32_t s = i % S, b = i % LOB;
            mbar_wait(smem_u32(&ready[b]), (i / LOB) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (lane == 0) {
                const uint32_t st = base + s * C::STAGE;
                const uint32_t alo = tmem + C::LO0 + b * BK;
#pragma unroll
                for (int k8 = 0; k8 < BK / 8; ++k8) {
                    const uint32_t ko = k8 * 1024;
                    const uint64_t da = smem_desc_mn128(st + C::AH + ko, C::SL);
                    const uint64_t dbh = smem_desc_mn128(st + C::BH + ko, C::SL);
                    mma_tf32(tmem, da, dbh, ID_SS, (i | (uint32_t)k8) ? 1u : 0u);  // [B_hi | B_lo]
                    mma_tf32_ts(tmem, alo + k8 * 8, dbh, ID_TS, 1u);
                }
                asm volatile(
                    "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                        smem_u32(&empty[s]))
                    : "memory");
                asm volatile(
                    "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                        smem_u32(&lofree[b]))
                    : "memory");
            }
            __syncwarp();
            if (!PROD && i >= 1) {
                const uint32_t j = i - 1;
                mbar_wait(smem_u32(&empty[j % S]), (j / S) & 1u);
                if (lane == 0 && j + S < nb) issue(j + S);
                __syncwarp();
            }
        }
    } else if (warp == 5) {
        if (PROD && lane == 0)
            for (uint32_t i = S; i < nb; ++i) {
                mbar_wait(smem_u32(&empty[(i - S) % S]), ((i - S) / S) & 1u);
                issue(i);
            }
    } else {
        const uint32_t lane_off = (warp * 32u) << 16;
        for (uint32_t i = 0; i < nb; ++i) {
            const uint32_t s = i % S, b = i % LOB;
            mbar_wait(smem_u32(&full[s]), (i / S) & 1u);
            if (i >= LOB) mbar_wait(smem_u32(&lofree[b]), ((i - LOB) / LOB) & 1u);  // MMA(i-LOB) read buffer b
            asm volatile("tcgen05.fence::after_thread_sync;");
            const unsigned char* st = base_p + s * C::STAGE;
            // A_lo of feature t (TMEM lane t), rows 0..BK-1 -> columns; warps past PS*32 own phantom lanes
            if (warp < (uint32_t)PS) {
                const unsigned char* sa = st + C::AH + warp * C::SL;
                const uint32_t c32 = lane / 8, w4 = (lane % 8) * 4;
#pragma unroll
                for (int k0 = 0; k0 < BK; k0 += 16) {
                    float lo[16];
#pragma unroll
                    for (int kk = 0; kk < 16; kk += 2) {
                        float x[2];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const uint32_t k = k0 + kk + h;
                            x[h] = *reinterpret_cast<const float*>(sa + (k / 4) * 512 + (k % 4) * 128 +
                                                                   ((c32 ^ (k % 4)) * 32) + w4);
                        }
                        const float2 l = lo_part2(x[0], x[1]);
                        lo[kk] = l.x, lo[kk + 1] = l.y;
                    }
                    tmem_st16(tmem + lane_off + C::LO0 + b * BK + k0, lo);
                }
            }
            if constexpr (QS == 0) {
                // B_lo of row k, 32-byte chunk j (columns 8j..8j+7) -> chunk j + 2 of the same row
                for (uint32_t f = t; f < 2u * BK; f += TM) {
                    const uint32_t k = f / 2, j = f % 2, row = (k / 4) * 512 + (k % 4) * 128;
                    const float4* src = reinterpret_cast<const float4*>(st + C::BH + row + ((j ^ (k % 4)) * 32));
                    float4* dst = reinterpret_cast<float4*>(const_cast<unsigned char*>(st) + C::BH + row +
                                                            (((j + 2) ^ (k % 4)) * 32));
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const float4 x = src[h];
                        const float2 l01 = lo_part2(x.x, x.y), l23 = lo_part2(x.z, x.w);
                        dst[h] = make_float4(l01.x, l01.y, l23.x, l23.y);
                    }
                }
            } else {
                // B_lo, elementwise at the same swizzled offsets
#pragma unroll
                for (uint32_t f = t; f < QS * (C::SL / 16); f += TM) {
                    const float4 x = reinterpret_cast<const float4*>(st + C::BH)[f];
                    const float2 l01 = lo_part2(x.x, x.y), l23 = lo_part2(x.z, x.w);
                    reinterpret_cast<float4*>(const_cast<unsigned char*>(st) + C::BL)[f] =
                        make_float4(l01.x, l01.y, l23.x, l23.y);
                }
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;");
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&ready[b])) : "memory");
        }
        // epilogue: TMEM lane t = feature t of A
        float* out = g.part + (size_t)blockIdx.x * g.p * g.q;
        if (nb == 0) {
            if (t < g.p)
                for (uint32_t j = 0; j < g.q; ++j) out[t * g.q + j] = 0.f;
        } else {
            const uint32_t last = nb - 1;
            mbar_wait(smem_u32(&lofree[last % LOB]), (last / LOB) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;");
            constexpr int HALF = (int)C::ND / 2;
            float acc[C::ND];
#pragma unroll
            for (int c = 0; c < (int)C::ND; c += 16) tmem_ld16(tmem + lane_off + (uint32_t)c, acc + c);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (t < g.p) {
#pragma unroll
                for (int j = 0; j < HALF; ++j)
                    if ((uint32_t)j < g.q) out[t * g.q + j] = acc[j] + acc[HALF + j];
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TCOLS));
}

// out[o] = sum over chunks c (in order) of part[c][o]: deterministic.
__global__ void k6_tn_reduce(const float* __restrict__ part, uint32_t chunks, uint32_t total, float* __restrict__ out) {
    const uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= total) return;
    float sum = 0.f;
    for (uint32_t c = 0; c < chunks; ++c) sum += part[(size_t)c * total + o];
    out[o] = sum;
}

bool make_map(CUtensorMap* map, const float* ptr, uint32_t cols, uint32_t rows, uint32_t box_rows,
              CUtensorMapSwizzle swz) {
    auto encode = tensor_map_encoder();
    if (!encode) return false;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    const cuuint32_t box[2] = {32, box_rows};
    const cuuint32_t es[2] = {1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int PS, int QS, int BK>
bool launch_tn_tc(gnna_ctx* ctx, const float* a, const float* b, uint32_t m, uint32_t p, uint32_t q, float* out) {
    CUtensorMap amap, bmap;
    if (!make_map(&amap, a, p, m, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) ||
        !make_map(&bmap, b, q, m, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
        return false;
    using C = TnCfg<PS, QS, BK>;
    {
    static const bool prod = [] {
        const char* e = std::getenv("GNNA_TN_PROD");  // A/B switch (0: the MMA warp refills)
        return !(e && *e == '0');
    }();
    auto kern = prod ? k6_gemm_tn_tc<PS, QS, BK, true> : k6_gemm_tn_tc<PS, QS, BK, false>;
    static std::atomic<uint64_t> attr{0};
    smem_attr_once(attr, kern, ctx->device, C::SMEM);
    const uint32_t nblk = (m + BK - 1) / BK;
    uint32_t ctas = nblk < (uint32_t)ctx->num_sms ? nblk : (uint32_t)ctx->num_sms;
    const uint32_t bpc = (nblk + ctas - 1) / ctas;
    ctas = (nblk + bpc - 1) / bpc;
    const uint32_t total = p * q;
    DevBuf<float> part((size_t)ctas * total, ctx->stream);
    TnArgs g{m, p, q, nblk, bpc, part.get()};
    kern<<<ctas, TN_THREADS + (prod ? 32 : 0), C::SMEM, ctx->stream>>>(amap, bmap, g);
    launched(ctx, "k6_gemm_tn_tc");
    static const bool seq = std::getenv("GNNA_TN_SEQ_REDUCE") != nullptr;  // A/B switch
    if (seq) {
        k6_tn_reduce<<<(total + 255) / 256, 256, 0, ctx->stream>>>(part.get(), ctas, total, out);
        launched(ctx, "k6_tn_reduce");
    } else {
        k_reduce_partials<<<(total + 31) / 32, 1024, 0, ctx->stream>>>(part.get(), ctas, total, out);
        launched(ctx, "k_reduce_partials");
    }
    return true;
    }
}

}  // namespace

// out = a(m x k) · w(k x n) [+ bias, relu | * row_scale] on tcgen05.  Returns
// false (nothing launched) for shapes this kernel does not take (k > 128).
bool gemm_tc_f32(gnna_ctx* ctx, const float* a, const float* w, const float* bias, const double* row_scale,
                 float* out, uint32_t m, uint32_t k, uint32_t n, int epilogue) {
    if (k == 0 || k > 128 || m == 0 || n == 0) return false;
    TcArgs g{a, w, bias, row_scale, out, m, k, n, epilogue, (m + TM - 1) / TM,
             (k % 4 == 0 && ((uintptr_t)a % 16 == 0)) ? 1 : 0, (k % 2 == 0 && ((uintptr_t)a % 8 == 0)) ? 1 : 0};
    static const bool no_tma = std::getenv("GNNA_GEMM_TC_LD") != nullptr;  // A/B switch
    if (g.vec && !no_tma) {
        const bool ok = k <= 32 ? launch_tma_n<32>(ctx, g)
                        : k <= 64 ? launch_tma_n<64>(ctx, g)
                        : k <= 96 ? launch_tma_n<96>(ctx, g)
                                  : launch_tma_n<128>(ctx, g);
        if (ok) return true;
    }
    if (k <= 16)
        launch_tc_n<16>(ctx, g);
    else if (k <= 32)
        launch_tc_n<32>(ctx, g);
    else if (k <= 64)
        launch_tc_n<64>(ctx, g);
    else if (k <= 96)
        launch_tc_n<96>(ctx, g);
    else
        launch_tc_n<128>(ctx, g);
    return true;
}

namespace {
template <int PS, int QS>
bool launch_tn_bk(gnna_ctx* ctx, const float* a, const float* b, uint32_t m, uint32_t p, uint32_t q, float* out) {
    static const bool big = [] {
        const char* e = std::getenv("GNNA_TN_BK");  // A/B switch (64: always 64-row blocks)
        return !(e && std::atoi(e) == 64);
    }();
    if constexpr (TnCfg<PS, QS, 128>::S >= 3)
        if (big) return launch_tn_tc<PS, QS, 128>(ctx, a, b, m, p, q, out);
    return launch_tn_tc<PS, QS, 64>(ctx, a, b, m, p, q, out);
}
}  // namespace

// out(p x q) = a(m x p)^T b(m x q) on tcgen05.  Returns false (nothing
// launched) unless p, q are multiples of 4 (TMA row pitch), p <= 128, q <= 64
// and both operands are 16-byte aligned.
bool gemm_tn_tc_f32(gnna_ctx* ctx, const float* a, const float* b, uint32_t m, uint32_t p, uint32_t q, float* out) {
    static const bool off = std::getenv("GNNA_GEMM_SIMT") != nullptr;  // A/B switch
    if (off || m == 0 || p == 0 || q == 0 || p > 128 || q > 64 || p % 4 || q % 4 || (uintptr_t)a % 16 ||
        (uintptr_t)b % 16)
        return false;
    const uint32_t ps = (p + 31) / 32;
    auto go = [&](auto qs) {
        constexpr int QS = decltype(qs)::value;
        switch (ps) {
            case 1: return launch_tn_bk<1, QS>(ctx, a, b, m, p, q, out);
            case 2: return launch_tn_bk<2, QS>(ctx, a, b, m, p, q, out);
            case 3: return launch_tn_bk<3, QS>(ctx, a, b, m, p, q, out);
            default: return launch_tn_bk<4, QS>(ctx, a, b, m, p, q, out);
        }
    };
    static const bool pack = [] {
        const char* e = std::getenv("GNNA_TN_PACK");  // A/B switch (0: separate B_lo slice)
        return !(e && *e == '0');
    }();
    if (q <= 16 && pack) return go(std::integral_constant<int, 0>{});
    return q <= 32 ? go(std::integral_constant<int, 1>{}) : go(std::integral_constant<int, 2>{});
}

}  // namespace gnna
