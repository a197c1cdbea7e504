// K3 / K3A / K4: neighbor aggregation for sm_100a.
//
// K3 (scheduled, engine.cpp:200-311): a team of TEAM lanes owns one workload
// unit (neighbor group).  Lanes split the row into 16-byte vectors (float4 /
// double2; the north star's "dimension workers"): lane t owns vector chunks
// t, t+TEAM, ... (Cyclic) or a contiguous block (Sequential).  A CTA holds
// whole schedule blocks (wpb units, Algorithm 1), so every run is CTA-local:
//   - a unit that is a whole run of a node living in one block stores its
//     partial straight to HBM (the common case once ngs >= degree);
//   - otherwise partials go to shared memory and the run's leader team sums
//     them in unit order (= the reference's slot accumulation) and flushes;
//   - a run of a node spanning several blocks is written to a carry slot and
//     the last CTA to write one of the node's carries adds them in block
//     order (carry_arrive); zero-degree rows are written by trailing blocks.
// The summation tree is the reference's: per unit, sequential over CSR
// order from 0; per run, sequential over units from 0; per node, sequential
// over blocks from 0.  In fp64 this makes the result bitwise equal to
// aggregate_scheduled; in fp32 it is the same tree in fp32.  No float
// atomics anywhere, so results are run-to-run deterministic.
//
// K4 (rows): one team per CSR row, CSR order (aggregate_oracle,
// engine.cpp:149-160), with exact fp64 variants of normalized_aggregate
// (engine.cpp:355-367) and the GIN self term (engine.cpp:394-400).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "gnna_common.cuh"

namespace {

using gnna::DevBuf;

template <class T, int VEC>
struct alignas(sizeof(T) * VEC) Vec {
    T a[VEC];
};

template <class T, int VEC>
__device__ __forceinline__ Vec<T, VEC> ldv(const T* p) {
    Vec<T, VEC> r;
    if constexpr (sizeof(T) * VEC == 16 && sizeof(T) == 4) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(p));
        r.a[0] = t.x; r.a[1] = t.y; r.a[2] = t.z; r.a[3] = t.w;
    } else if constexpr (sizeof(T) * VEC == 16 && sizeof(T) == 8) {
        const double2 t = __ldg(reinterpret_cast<const double2*>(p));
        r.a[0] = t.x; r.a[1] = t.y;
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i) r.a[i] = __ldg(p + i);
    }
    return r;
}

template <class T, int VEC>
__device__ __forceinline__ void stv(T* p, const Vec<T, VEC>& v) {
    if constexpr (sizeof(T) * VEC == 16 && sizeof(T) == 4) {
        __stcs(reinterpret_cast<float4*>(p), make_float4(v.a[0], v.a[1], v.a[2], v.a[3]));
    } else if constexpr (sizeof(T) * VEC == 16 && sizeof(T) == 8) {
        __stcs(reinterpret_cast<double2*>(p), make_double2(v.a[0], v.a[1]));
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i) p[i] = v.a[i];
    }
}

// One row vector to the NVLS multicast address of a replicated y: the
// NVSwitch writes it into every rank's copy (multimem.st, sm_90+).
template <class T, int VEC>
__device__ __forceinline__ void stv_multimem(T* p, const Vec<T, VEC>& v) {
    if constexpr (sizeof(T) == 4 && VEC == 4) {
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.a[0]),
                     "f"(v.a[1]), "f"(v.a[2]), "f"(v.a[3])
                     : "memory");
    } else if constexpr (sizeof(T) == 4) {
#pragma unroll
        for (int i = 0; i < VEC; ++i)
            asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p + i), "f"(v.a[i]) : "memory");
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i)
            asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p + i), "d"(v.a[i]) : "memory");
    }
}

template <class T, int VEC>
__device__ __forceinline__ void vzero(Vec<T, VEC>& v) {
#pragma unroll
    for (int i = 0; i < VEC; ++i) v.a[i] = T(0);
}

// acc += v, one IEEE add per element (never contracted: no multiply).
template <class T, int VEC>
__device__ __forceinline__ void vadd(Vec<T, VEC>& acc, const Vec<T, VEC>& v) {
#pragma unroll
    for (int i = 0; i < VEC; ++i) acc.a[i] = acc.a[i] + v.a[i];
}

__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }

// acc += c * v with a separately rounded product (the reference's
// `out[d] += c * in[d]` compiled without FMA contraction).
template <class T, int VEC>
__device__ __forceinline__ void vaxpy_rn(Vec<T, VEC>& acc, T c, const Vec<T, VEC>& v) {
#pragma unroll
    for (int i = 0; i < VEC; ++i) acc.a[i] = add_rn(acc.a[i], mul_rn(c, v.a[i]));
}

enum : uint32_t { EPI_SCALE = 1, EPI_SELF = 2, EPI_RELU = 4, EPI_MASK = 8 };

struct AggArgs {
    // schedule
    const uint64_t* part_ptr;
    const uint32_t* part2node;
    const uint8_t* uflags;
    const uint32_t* cidx;
    uint64_t units;    // K3: plan units; K4: rows
    uint32_t upc;      // units per CTA
    uint32_t r0;       // K4: first row
    const uint64_t* row_ptr;
    const uint32_t* col;
    const void* x;
    void* y;
    const void* xself;  // EPI_SELF reads x[v] here when set (x is then the pre-scaled gather source)
    void* carry;
    uint32_t dim, nvec, kpl;
    int seq;
    // epilogue (final writes only)
    uint32_t epi;
    const float* scale;   // EPI_SCALE: per-row multiplier (fp32 GCN fold)
    double alpha;         // EPI_SELF:  y += alpha * x[v]  (or sw[v] * x[v] when sw != null)
    const float* sw;      // EPI_SELF per-node self weights (GCN: norm[v] if v gets an implicit loop, else 0)
    const void* mask;     // EPI_MASK: y[v][d] = mask[v][d] > 0 ? y[v][d] : 0 (ReLU backward)
    const float* nw;      // per-source-node weights (fp32 path): acc += nw[u] * x[u], u = col[e]
    // fused all-gather: final row values also go to the peer
    // replicas of y (P2P stores over NVLink), or, when mc is set, only to the
    // NVLS multicast address of the replicated y (every rank's copy, self included)
    void* peers[GNNA_MAX_PEERS];
    uint32_t npeer;
    void* mc;
    // look-ahead: CTA k prefetches into L2 the unit metadata of CTA k + pf
    // (the CTA that takes its slot when it retires); 0 = off
    uint32_t pf;
    // fused carry combine / empty rows (formerly the K3b pass)
    const uint32_t* carry_split;  // carry slot -> split-node index
    uint32_t* split_cnt;          // per split node: carries written so far this launch (reset by the last)
    const uint32_t* split_node;   // per split node: node id
    const uint32_t* split_first;  // per split node: first carry slot
    const uint32_t* split_count;  // per split node: carry slots
    const uint32_t* empty_rows;   // zero-degree rows of the range
    uint64_t nempty;
    uint64_t unit_blocks;         // CTAs that own units; blocks past them write empty rows
    // K4 exact modes
    const double* norm;
    const uint8_t* self;
};

template <class T, int VEC, int TEAM, int KMAX>
struct Lanes {
    uint32_t off[KMAX];
    bool ok[KMAX];
    __device__ __forceinline__ void init(const AggArgs& a, uint32_t lane, uint32_t k0) {
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const uint32_t kk = k0 + k;
            const uint32_t c = a.seq ? lane * a.kpl + kk : lane + kk * TEAM;
            ok[k] = kk < a.kpl && c < a.nvec;
            off[k] = c * VEC;
        }
    }
};

// Per-row epilogue scalars are prefetched into L1 when the row's unit starts
// (K3), so the final store's loads hit L1 instead of trailing the gather by
// an L2 round trip; no registers are held across the gather.
__device__ __forceinline__ void prefetch_l1(const void* p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

template <class T, int VEC, bool FAN = false>
__device__ __forceinline__ void store_final(const AggArgs& a, uint32_t v, uint32_t off, Vec<T, VEC> val) {
    T* y = static_cast<T*>(a.y) + (size_t)v * a.dim + off;
    if (a.epi) {
        if (a.epi & EPI_SELF) {
            const T c = a.sw ? T(a.sw[v]) : T(a.alpha);
            if (c != T(0)) {
                const Vec<T, VEC> xv =
                    ldv<T, VEC>(static_cast<const T*>(a.xself ? a.xself : a.x) + (size_t)v * a.dim + off);
                vaxpy_rn(val, c, xv);
            }
        }
        if (a.epi & EPI_SCALE) {
            const T s = T(a.scale[v]);
#pragma unroll
            for (int i = 0; i < VEC; ++i) val.a[i] = s * val.a[i];
        }
        if (a.epi & EPI_RELU) {
#pragma unroll
            for (int i = 0; i < VEC; ++i) val.a[i] = val.a[i] > T(0) ? val.a[i] : T(0);
        }
        if (a.epi & EPI_MASK) {
            const Vec<T, VEC> m = ldv<T, VEC>(static_cast<const T*>(a.mask) + (size_t)v * a.dim + off);
#pragma unroll
            for (int i = 0; i < VEC; ++i) val.a[i] = m.a[i] > T(0) ? val.a[i] : T(0);
        }
    }
    if constexpr (FAN) {  // separate instantiations: the register-capped default K3 is untouched
        if (a.mc) {
            stv_multimem<T, VEC>(static_cast<T*>(a.mc) + (size_t)v * a.dim + off, val);
            return;
        }
        stv<T, VEC>(y, val);
        for (uint32_t i = 0; i < a.npeer; ++i)
            stv<T, VEC>(static_cast<T*>(a.peers[i]) + (size_t)v * a.dim + off, val);
    } else {
        stv<T, VEC>(y, val);
    }
}


// Occupancy vs. loads-in-flight, measured on B200 (profiles/README.md):
// register-capped occupancy beats deep unrolling.  Every plain gather runs 6
// row vectors in flight per lane at <= 64 registers (4 CTAs of 256 threads
// per SM): the r01m small-team A/B on C3 (d = 16) measured UNR/minb 6/4 at
// 0.0563 ms against 8/3 at 0.0645 ms (4/5: 0.0625, 4/6: 0.079, 8/4: 0.073).
// The per-source-weight gather (EW) on narrow teams holds one more value per
// row vector and spills at 64 registers, so it keeps 8 in flight at <= 80
// registers (3 CTAs): 0.080 vs 0.095 ms.  GNNA_K3_UNR / GNNA_K3_MINB (all
// teams) and GNNA_K3_UNR_S / GNNA_K3_MINB_S (plain narrow teams) override for
// experiment builds (`make variants`).
template <int TEAM, int KMAX, bool EW = false>
struct K3Tune {
#ifndef GNNA_K3_UNR_S
#define GNNA_K3_UNR_S 6
#endif
#ifndef GNNA_K3_MINB_S
#define GNNA_K3_MINB_S 4
#endif
#ifndef GNNA_K3_UNR_W
#define GNNA_K3_UNR_W 6
#endif
#ifndef GNNA_K3_MINB_W
#define GNNA_K3_MINB_W 4
#endif
#ifdef GNNA_K3_UNR
    static constexpr int unr1 = GNNA_K3_UNR;
#else
    static constexpr int unr1 = TEAM >= 8 ? GNNA_K3_UNR_W : (EW ? 8 : GNNA_K3_UNR_S);
#endif
#ifdef GNNA_K3_MINB
    static constexpr int minb = GNNA_K3_MINB;
#else
    static constexpr int minb = TEAM >= 8 ? GNNA_K3_MINB_W : (EW ? 3 : GNNA_K3_MINB_S);
#endif
    static constexpr int unr = KMAX == 1 ? unr1 : (KMAX == 2 ? (unr1 + 1) / 2 : (unr1 + 3) / 4);
#ifdef GNNA_K3_BATCH
    static constexpr int batch = TEAM >= 8 ? 32 : GNNA_K3_BATCH;
#else
    static constexpr int batch = 32;
#endif
};

// Team-cooperative gather over [b, e) into acc: every output dimension is a
// sequential sum in CSR order from 0 (engine.cpp:237-240).  The warp walks its teams' neighbour
// lists in batches of 32 CSR entries: one coalesced index load per batch
// (each lane holds 32/TEAM indices), indices are broadcast inside the team
// with width-TEAM shuffles, and UNR x KMAX 16-byte row vectors per lane are
// in flight before the in-order adds.  Loop bounds are warp-uniform (max
// over the warp's teams), loads/adds of finished teams are predicated off.
// EW (fp32 path): per-SOURCE-node weights nw[u] (GCN: norm[u]) gathered
// beside the row vectors, acc += nw[col[e]] * x[col[e]] (one FMA per
// element).  The weight load depends only on the index, so it issues with the
// row loads (no extra latency level) and keeps nothing live across a batch.
template <class T, int VEC, int TEAM, int KMAX, bool EW = false>
__device__ __forceinline__ void gather_team(const AggArgs& a, uint64_t b, uint64_t e, uint32_t lane,
                                            const uint32_t (&off)[KMAX], const bool (&ok)[KMAX],
                                            Vec<T, VEC> (&acc)[KMAX]) {
    constexpr int UNR = K3Tune<TEAM, KMAX, EW>::unr;
    constexpr int BATCH = K3Tune<TEAM, KMAX, EW>::batch;  // CSR entries per index batch
    constexpr int R = BATCH / TEAM;                    // indices held per lane per batch
    const T* __restrict__ x = static_cast<const T*>(a.x);
    const uint32_t* __restrict__ col = a.col;
    const uint32_t len = (uint32_t)(e - b);
    const uint32_t wlen = __reduce_max_sync(0xffffffffu, len);
    // (A/B, r01: gathering the batch's weights once per lane and shuffling
    // them like the indices spills on wide teams: C5 25.5 vs 17.6 ms.)
    for (uint32_t base = 0; base < wlen; base += BATCH) {
        uint32_t idxr[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t j = base + lane + r * TEAM;
            idxr[r] = j < len ? __ldg(col + b + j) : 0u;
        }
        const uint32_t cnt = len > base ? min((uint32_t)BATCH, len - base) : 0u;
        const uint32_t wcnt = __reduce_max_sync(0xffffffffu, cnt);
#pragma unroll
        for (int q0 = 0; q0 < BATCH; q0 += UNR) {
            if ((uint32_t)q0 >= wcnt) break;
            uint32_t idx[UNR];
            float wgt[EW ? UNR : 1];
#pragma unroll
            for (int u = 0; u < UNR; ++u) idx[u] = __shfl_sync(0xffffffffu, idxr[(q0 + u) / TEAM], (q0 + u) % TEAM, TEAM);
            Vec<T, VEC> val[UNR][KMAX];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                if constexpr (EW) wgt[u] = (uint32_t)(q0 + u) < cnt ? __ldg(a.nw + idx[u]) : 0.f;
#pragma unroll
                for (int k = 0; k < KMAX; ++k)
                    if (ok[k] && (uint32_t)(q0 + u) < cnt)
                        val[u][k] = ldv<T, VEC>(x + (size_t)idx[u] * a.dim + off[k]);
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u)
#pragma unroll
                for (int k = 0; k < KMAX; ++k)
                    if (ok[k] && (uint32_t)(q0 + u) < cnt) {
                        if constexpr (EW) {
#pragma unroll
                            for (int i = 0; i < VEC; ++i) acc[k].a[i] = fmaf(wgt[u], val[u][k].a[i], acc[k].a[i]);
                        } else {
                            vadd(acc[k], val[u][k]);
                        }
                    }
        }
    }
}

// A split node's carries (its runs' partials, one per schedule block it
// spans) are combined by whichever CTA writes the LAST of them: each writer
// fences and counts; the last one sums the node's carries in block order
// (= the reference's flush order, engine.cpp:294-308) and applies the final
// store.  Deterministic whatever the arrival order, and no second pass.
template <class T, int VEC, int TEAM, bool FAN>
__device__ __forceinline__ void carry_arrive(const AggArgs& a, uint32_t c, uint32_t lane) {
    const uint32_t wl = threadIdx.x & 31;
    const uint32_t tmask = (TEAM == 32 ? 0xffffffffu : ((1u << TEAM) - 1u)) << (wl - lane);
    __threadfence();  // this lane's carry stores, before the count
    __syncwarp(tmask);
    uint32_t last = 0, k = 0;
    if (lane == 0) {
        k = __ldg(a.carry_split + c);
        last = atomicAdd(a.split_cnt + k, 1u) + 1u == __ldg(a.split_count + k) ? 1u : 0u;
    }
    last = __shfl_sync(tmask, last, 0, TEAM);
    if (!last) return;
    k = __shfl_sync(tmask, k, 0, TEAM);
    __threadfence();  // every other writer's carries are visible (they fenced before counting)
    const uint32_t first = __ldg(a.split_first + k), cnt = __ldg(a.split_count + k), v = __ldg(a.split_node + k);
    const T* cy = static_cast<const T*>(a.carry) + (size_t)first * a.dim;
    for (uint32_t ch = lane; ch < a.nvec; ch += TEAM) {
        Vec<T, VEC> acc;
        vzero(acc);
        for (uint32_t j = 0; j < cnt; ++j) {
            const T* p = cy + (size_t)j * a.dim + ch * VEC;
            Vec<T, VEC> t;
#pragma unroll
            for (int i = 0; i < VEC; ++i) t.a[i] = __ldcg(p + i);  // L2: written by other CTAs
            vadd(acc, t);
        }
        store_final<T, VEC, FAN>(a, v, ch * VEC, acc);
    }
    if (lane == 0) a.split_cnt[k] = 0;  // ready for the next launch (stream-ordered)
}

// Blocks past the unit blocks: zero-degree rows get the epilogue of an empty sum.
template <class T, int VEC, int TEAM, bool FAN>
__device__ __forceinline__ void empty_rows_block(const AggArgs& a) {
    const uint32_t tu = threadIdx.x / TEAM, lane = threadIdx.x % TEAM;
    const uint64_t i = (blockIdx.x - a.unit_blocks) * (uint64_t)(blockDim.x / TEAM) + tu;
    if (i >= a.nempty) return;
    const uint32_t v = __ldg(a.empty_rows + i);
    Vec<T, VEC> z;
    vzero(z);
    for (uint32_t ch = lane; ch < a.nvec; ch += TEAM) store_final<T, VEC, FAN>(a, v, ch * VEC, z);
}

// Wide-row plans (TEAM > 8 or KMAX > 1): split nodes add their carries in
// block order in a second launch (one team per node).
template <class T, int VEC, int TEAM, bool FAN>
__global__ void __launch_bounds__(256) k3b_split(AggArgs a, uint64_t nsplit) {
    const uint32_t tu = threadIdx.x / TEAM, lane = threadIdx.x % TEAM;
    const uint64_t k = (uint64_t)blockIdx.x * (256 / TEAM) + tu;
    if (k >= nsplit) return;
    const uint32_t v = a.split_node[k], first = a.split_first[k], cnt = a.split_count[k];
    const T* cy = static_cast<const T*>(a.carry) + (size_t)first * a.dim;
    for (uint32_t ch = lane; ch < a.nvec; ch += TEAM) {
        Vec<T, VEC> acc;
        vzero(acc);
        for (uint32_t j = 0; j < cnt; ++j) vadd(acc, ldv<T, VEC>(cy + (size_t)j * a.dim + ch * VEC));
        store_final<T, VEC, FAN>(a, v, ch * VEC, acc);
    }
}

// ----------------------------------------------------------------- K3 ---
template <class T, int VEC, int TEAM, int KMAX, bool EW, bool FAN = false>
__global__ void __launch_bounds__(256, K3Tune<TEAM, KMAX, EW>::minb) k3_aggregate(AggArgs a) {
    using VT = Vec<T, VEC>;
    if (blockIdx.x >= a.unit_blocks) {  // block-uniform: no barrier is skipped by part of a CTA
        empty_rows_block<T, VEC, TEAM, FAN>(a);
        return;
    }
    extern __shared__ __align__(16) unsigned char smem_raw[];
    VT* sm = reinterpret_cast<VT*>(smem_raw);  // [upc][KMAX][TEAM]
    const uint32_t tu = threadIdx.x / TEAM, lane = threadIdx.x % TEAM;
    const uint64_t u = (uint64_t)blockIdx.x * a.upc + tu;
    const bool active = tu < a.upc && u < a.units;
    uint64_t b = 0, e = 0;
    uint32_t v = 0;
    uint8_t f = 0;
    if (active) {
        b = __ldg(a.part_ptr + u);
        e = __ldg(a.part_ptr + u + 1);
        v = __ldg(a.part2node + u);
        f = __ldg(a.uflags + u);
    }
    if (active && a.epi) {
        if (a.epi & EPI_SCALE) prefetch_l1(a.scale + v);
        if ((a.epi & EPI_SELF) && a.sw) prefetch_l1(a.sw + v);
    }
    if (a.pf && threadIdx.x < 32) {  // fire-and-forget: nothing waits on these
        const uint64_t f0 = ((uint64_t)blockIdx.x + a.pf) * a.upc;
        if (f0 < a.units) {
            const uint32_t l = threadIdx.x;
            const uint64_t cnt = a.units - f0 < (uint64_t)a.upc ? a.units - f0 : (uint64_t)a.upc;
            if ((uint64_t)l * 16 <= cnt) prefetch_l2(a.part_ptr + f0 + (uint64_t)l * 16);   // 128 B = 16 x u64
            if ((uint64_t)l * 32 < cnt) prefetch_l2(a.part2node + f0 + (uint64_t)l * 32);  // 128 B = 32 x u32
            if ((uint64_t)l * 128 < cnt) prefetch_l2(a.uflags + f0 + (uint64_t)l * 128);
        }
    }
    const bool direct = (f & (UF_LEADER | UF_RUN_END)) == (UF_LEADER | UF_RUN_END) && !(f & UF_SPLIT);
    const bool staged = active && !direct;
    const bool need_smem = __syncthreads_or(staged);
    for (uint32_t k0 = 0; k0 < a.kpl; k0 += KMAX) {
        Lanes<T, VEC, TEAM, KMAX> L;
        L.init(a, lane, k0);
        VT acc[KMAX];
#pragma unroll
        for (int k = 0; k < KMAX; ++k) vzero(acc[k]);
        gather_team<T, VEC, TEAM, KMAX, EW>(a, b, e, lane, L.off, L.ok, acc);  // all lanes (b = e for idle teams)
        if (active && direct) {
#pragma unroll
            for (int k = 0; k < KMAX; ++k)
                if (L.ok[k]) store_final<T, VEC, FAN>(a, v, L.off[k], acc[k]);
        }
        if (need_smem) {
            if (staged) {
#pragma unroll
                for (int k = 0; k < KMAX; ++k) sm[(tu * KMAX + k) * TEAM + lane] = acc[k];
            }
            __syncthreads();
            if (staged && (f & UF_LEADER)) {
                VT r[KMAX];
#pragma unroll
                for (int k = 0; k < KMAX; ++k) vzero(r[k]);
                uint32_t t2 = tu;
                uint8_t f2 = f;
                for (;;) {
#pragma unroll
                    for (int k = 0; k < KMAX; ++k) vadd(r[k], sm[(t2 * KMAX + k) * TEAM + lane]);
                    if (f2 & UF_RUN_END) break;
                    ++t2;
                    f2 = __ldg(a.uflags + u + (t2 - tu));
                }
                if (f & UF_SPLIT) {
                    T* cy = static_cast<T*>(a.carry) + (size_t)__ldg(a.cidx + u) * a.dim;
#pragma unroll
                    for (int k = 0; k < KMAX; ++k)
                        if (L.ok[k]) stv<T, VEC>(cy + L.off[k], r[k]);
                    // rows of 16+ vectors leave the combine to k3b_split: inlining it
                    // there costs the gather loop registers (same-box A/B, C4: fp32
                    // 0.0513 -> 0.0533 ms, fp64 0.084 -> 0.094 ms), while for narrow
                    // rows the saved launch wins (C3 0.0563 -> 0.0521 ms)
                    if constexpr (KMAX == 1 && TEAM <= 8) carry_arrive<T, VEC, TEAM, FAN>(a, __ldg(a.cidx + u), lane);
                } else {
#pragma unroll
                    for (int k = 0; k < KMAX; ++k)
                        if (L.ok[k]) store_final<T, VEC, FAN>(a, v, L.off[k], r[k]);
                }
            }
            __syncthreads();
        }
    }
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- K3A ---
// K3 with the row gather landing in shared memory (cp.async, 16 B per lane
// per row) instead of registers, for narrow rows (one chunk per lane).  The
// plain K3 holds its in-flight rows in registers, so memory-level
// parallelism is capped by the 64-register budget that buys 4 CTAs per SM
// (6 rows in flight per lane); ncu (r02) shows it latency-bound on exactly
// those gathers and on the index loads.  Here a lane issues up to K3A_ROWS
// cp.async row copies into its own smem slots, waits once, then adds the
// rows in CSR order from shared memory, so the summation tree is unchanged
// (fp64 bitwise) while rows in flight per lane grow 2-3x at fewer registers
// (occupancy is now set by shared memory).
#ifndef K3A_ROWS
#define K3A_ROWS 12
#endif
#ifndef K3A_MINB
#define K3A_MINB 5
#endif

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// buf: this warp's slots, row q of lane wl at buf[q * 32 + wl].
template <class T, int VEC, int TEAM, bool EW>
__device__ __forceinline__ void gather_async(const AggArgs& a, uint64_t b, uint64_t e, uint32_t lane, uint32_t off,
                                             bool ok, Vec<T, VEC>& acc, Vec<T, VEC>* buf) {
    constexpr int ROWS = K3A_ROWS;
    constexpr int R = 32 / TEAM;  // indices held per lane per 32-entry batch
    const T* __restrict__ x = static_cast<const T*>(a.x);
    const uint32_t wl = threadIdx.x & 31;
    const uint32_t len = (uint32_t)(e - b);
    const uint32_t wlen = __reduce_max_sync(0xffffffffu, len);
    for (uint32_t base = 0; base < wlen; base += 32) {
        uint32_t idxr[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t j = base + lane + r * TEAM;
            idxr[r] = j < len ? __ldg(a.col + b + j) : 0u;
        }
        const uint32_t cnt = len > base ? min(32u, len - base) : 0u;
        const uint32_t wcnt = __reduce_max_sync(0xffffffffu, cnt);
#pragma unroll
        for (int q0 = 0; q0 < 32; q0 += ROWS) {  // unrolled: idxr[] indices are compile-time (registers)
            if ((uint32_t)q0 >= wcnt) break;
            float wgt[EW ? ROWS : 1];
#pragma unroll
            for (int u = 0; u < ROWS; ++u) {
                const uint32_t q = q0 + u;
                if (q0 + u < 32) {
                    uint32_t idx = __shfl_sync(0xffffffffu, idxr[(q0 + u) / TEAM], (q0 + u) % TEAM, TEAM);
                    if constexpr (EW) wgt[u] = q < cnt ? __ldg(a.nw + idx) : 0.f;
                    if (ok && q < cnt) cp_async16(smem_addr(&buf[u * 32 + wl]), x + (size_t)idx * a.dim + off);
                }
            }
            cp_async_wait_all();
#pragma unroll
            for (int u = 0; u < ROWS; ++u) {
                if (ok && (uint32_t)(q0 + u) < cnt) {
                    const Vec<T, VEC> v = buf[u * 32 + wl];
                    if constexpr (EW) {
#pragma unroll
                        for (int i = 0; i < VEC; ++i) acc.a[i] = fmaf(wgt[u], v.a[i], acc.a[i]);
                    } else {
                        vadd(acc, v);
                    }
                }
            }
        }
    }
}

template <class T, int VEC, int TEAM, bool EW, bool FAN = false>
__global__ void __launch_bounds__(256, K3A_MINB) k3a_aggregate(AggArgs a) {
    using VT = Vec<T, VEC>;
    if (blockIdx.x >= a.unit_blocks) {
        empty_rows_block<T, VEC, TEAM, FAN>(a);
        return;
    }
    extern __shared__ __align__(16) unsigned char smem_raw[];
    VT* sm = reinterpret_cast<VT*>(smem_raw);   // [upc][TEAM] staged partials
    VT* gbuf = sm + blockDim.x + (threadIdx.x / 32) * (K3A_ROWS * 32);  // this warp's gather slots
    const uint32_t tu = threadIdx.x / TEAM, lane = threadIdx.x % TEAM;
    const uint64_t u = (uint64_t)blockIdx.x * a.upc + tu;
    const bool active = tu < a.upc && u < a.units;
    uint64_t b = 0, e = 0;
    uint32_t v = 0;
    uint8_t f = 0;
    if (active) {
        b = __ldg(a.part_ptr + u);
        e = __ldg(a.part_ptr + u + 1);
        v = __ldg(a.part2node + u);
        f = __ldg(a.uflags + u);
    }
    if (active && a.epi) {
        if (a.epi & EPI_SCALE) prefetch_l1(a.scale + v);
        if ((a.epi & EPI_SELF) && a.sw) prefetch_l1(a.sw + v);
    }
    if (a.pf && threadIdx.x < 32) {  // metadata look-ahead, as in K3
        const uint64_t f0 = ((uint64_t)blockIdx.x + a.pf) * a.upc;
        if (f0 < a.units) {
            const uint32_t l = threadIdx.x;
            const uint64_t cnt = a.units - f0 < (uint64_t)a.upc ? a.units - f0 : (uint64_t)a.upc;
            if ((uint64_t)l * 16 <= cnt) prefetch_l2(a.part_ptr + f0 + (uint64_t)l * 16);
            if ((uint64_t)l * 32 < cnt) prefetch_l2(a.part2node + f0 + (uint64_t)l * 32);
            if ((uint64_t)l * 128 < cnt) prefetch_l2(a.uflags + f0 + (uint64_t)l * 128);
        }
    }
    const bool direct = (f & (UF_LEADER | UF_RUN_END)) == (UF_LEADER | UF_RUN_END) && !(f & UF_SPLIT);
    const bool staged = active && !direct;
    const bool need_smem = __syncthreads_or(staged);
    const uint32_t off = lane * VEC;
    const bool ok = lane < a.nvec;
    VT acc;
    vzero(acc);
    gather_async<T, VEC, TEAM, EW>(a, b, e, lane, off, ok, acc, gbuf);
    if (active && direct && ok) store_final<T, VEC, FAN>(a, v, off, acc);
    if (need_smem) {
        if (staged) sm[tu * TEAM + lane] = acc;
        __syncthreads();
        if (staged && (f & UF_LEADER)) {
            VT r;
            vzero(r);
            uint32_t t2 = tu;
            uint8_t f2 = f;
            for (;;) {
                vadd(r, sm[t2 * TEAM + lane]);
                if (f2 & UF_RUN_END) break;
                ++t2;
                f2 = __ldg(a.uflags + u + (t2 - tu));
            }
            if (f & UF_SPLIT) {
                const uint32_t c = __ldg(a.cidx + u);
                if (ok) stv<T, VEC>(static_cast<T*>(a.carry) + (size_t)c * a.dim + off, r);
                carry_arrive<T, VEC, TEAM, FAN>(a, c, lane);
            } else if (ok) {
                store_final<T, VEC, FAN>(a, v, off, r);
            }
        }
    }
}

// ----------------------------------------------------------------- K4 ---
// MODE 0: plain CSR-order sum.  MODE 1: exact normalized_aggregate (per-edge
// c = norm[v]*norm[u], separately rounded c*x, implicit self loop last).
// MODE 2: exact GIN input (CSR-order sum, then + alpha*x[v]).
template <class T, int VEC, int TEAM, int KMAX, int MODE>
__global__ void __launch_bounds__(256, K3Tune<TEAM, KMAX>::minb) k4_rows(AggArgs a) {
    using VT = Vec<T, VEC>;
    const uint32_t tu = threadIdx.x / TEAM, lane = threadIdx.x % TEAM;
    const uint64_t i = (uint64_t)blockIdx.x * (256 / TEAM) + tu;
    const bool active = i < a.units;  // no early exit: gather_team is warp-collective
    const uint32_t v = active ? a.r0 + (uint32_t)i : 0u;
    const uint64_t b = active ? __ldg(a.row_ptr + v) : 0, e = active ? __ldg(a.row_ptr + v + 1) : 0;
    const T* __restrict__ x = static_cast<const T*>(a.x);
    for (uint32_t k0 = 0; k0 < a.kpl; k0 += KMAX) {
        Lanes<T, VEC, TEAM, KMAX> L;
        L.init(a, lane, k0);
        VT acc[KMAX];
#pragma unroll
        for (int k = 0; k < KMAX; ++k) vzero(acc[k]);
        if constexpr (MODE == 1) {
            const double nv = a.norm[v];
            for (uint64_t p = b; p < e; ++p) {
                const uint32_t uu = __ldg(a.col + p);
                const T c = T(__dmul_rn(nv, a.norm[uu]));
#pragma unroll
                for (int k = 0; k < KMAX; ++k)
                    if (L.ok[k]) vaxpy_rn(acc[k], c, ldv<T, VEC>(x + (size_t)uu * a.dim + L.off[k]));
            }
            if (active && a.self && a.self[v]) {
                const T c = T(__dmul_rn(nv, nv));
#pragma unroll
                for (int k = 0; k < KMAX; ++k)
                    if (L.ok[k]) vaxpy_rn(acc[k], c, ldv<T, VEC>(x + (size_t)v * a.dim + L.off[k]));
            }
        } else {
            gather_team<T, VEC, TEAM, KMAX>(a, b, e, lane, L.off, L.ok, acc);
            if constexpr (MODE == 2) {
#pragma unroll
                for (int k = 0; k < KMAX; ++k)
                    if (active && L.ok[k]) vaxpy_rn(acc[k], T(a.alpha), ldv<T, VEC>(x + (size_t)v * a.dim + L.off[k]));
            }
        }
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
            if (active && L.ok[k]) store_final<T, VEC>(a, v, L.off[k], acc[k]);
    }
}

// ----------------------------------------------------------- dispatch ---
uint32_t pow2ceil(uint32_t v) {
    uint32_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

uint32_t pow2floor(uint32_t v) {
    uint32_t p = 1;
    while (p * 2 <= v) p <<= 1;
    return p;
}

struct Shape {
    int vec;
    uint32_t team, kpl, kmax;
};

Shape choose_shape(int elem, uint32_t dim, uint32_t dw, uint32_t team_cap, const void* x, const void* y,
                   bool others_aligned = true) {
    Shape s;
    const int full = 16 / elem;
    // every row-vector operand (x, y, and the mask / peer replicas / multicast
    // address when present) must be 16-byte aligned for the vector path
    const bool aligned = ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0) && others_aligned;
    s.vec = (dim % full == 0 && aligned) ? full : 1;
    const uint32_t nvec = dim / s.vec;
    // The physical lane map is free: every output dimension is summed in the
    // same order whatever lane owns it.  By default a team spans the whole
    // row in 16-byte vectors (up to a warp); GNNA_K3_DW_TEAMS=1 restores the
    // literal map (dw scalar dimension workers = dw/vec vector lanes).
    static const bool dw_teams = std::getenv("GNNA_K3_DW_TEAMS") != nullptr;
    uint32_t t = dw_teams ? pow2ceil((dw + s.vec - 1) / s.vec) : 32u;
    t = std::min<uint32_t>(t, pow2ceil(nvec));
    t = std::min<uint32_t>(t, team_cap);
    static const int team_max = std::getenv("GNNA_K3_TEAM_MAX") ? std::atoi(std::getenv("GNNA_K3_TEAM_MAX")) : 0;
    if (team_max > 0) t = std::min<uint32_t>(t, (uint32_t)team_max);  // A/B: narrower teams, more units per warp
    t = std::max<uint32_t>(t, 1);
    s.team = std::min<uint32_t>(t, 32);
    s.kpl = (nvec + s.team - 1) / s.team;
    s.kmax = s.kpl <= 1 ? 1 : (s.kpl <= 2 ? 2 : 4);
    // fp64 rows of 4+ chunks per lane: two passes of KMAX 2 instead of one of
    // KMAX 4, whose 8 double2 accumulators + row vectors spill at the 64-register
    // cap (GNNA_K3_F64_KMAX4=1 restores one pass for A/B)
    static const bool f64_k4 = std::getenv("GNNA_K3_F64_KMAX4") != nullptr;
    if (elem == 8 && s.kmax == 4 && !f64_k4) s.kmax = 2;
    return s;
}

// K3A launch (cp.async row gather into shared memory): true when it ran.
template <class T, int VEC, int TEAM, bool EW, bool FAN>
void launch_k3a_v(gnna_ctx* ctx, AggArgs& a, uint64_t grid, unsigned threads) {
    auto kern = k3a_aggregate<T, VEC, TEAM, EW, FAN>;
    const size_t smem = (threads + (threads / 32) * K3A_ROWS * 32) * sizeof(Vec<T, VEC>);
    static bool attr = false;
    if (!attr) {  // the 256-thread size bounds every smaller one
        GNNA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)((256 + 8 * K3A_ROWS * 32) * sizeof(Vec<T, VEC>))));
        attr = true;
    }
    kern<<<(unsigned)grid, threads, smem, ctx->stream>>>(a);
    gnna::launched(ctx, "k3a_aggregate");
}

// K3A is used for narrow fp64 rows (one 16-byte chunk per lane): there the
// plain K3's register-held gather caps rows in flight (r02 A/B, C3 fp64:
// 0.081 vs 0.109 ms); narrow fp32 rows measured even (0.0563 both) and the
// weighted gather slower (0.094 vs 0.079), so fp32 keeps K3.  GNNA_K3A=0/2
// forces K3 / K3A everywhere it applies (A/B).
template <class T, int VEC, int TEAM>
bool k3a_applies(const AggArgs& a, uint32_t kmax) {
    if constexpr (TEAM >= 2 && TEAM <= 8 && sizeof(T) * VEC == 16) {
        static const int mode = std::getenv("GNNA_K3A") ? std::atoi(std::getenv("GNNA_K3A")) : 1;
        if (mode == 0 || kmax != 1 || a.kpl != 1 || a.upc * TEAM > 256) return false;
        if (a.nw && (a.npeer || a.mc)) return false;
        return mode == 2 || std::is_same<T, double>::value;
    } else {
        (void)a; (void)kmax;
        return false;
    }
}

template <class T, int VEC, int TEAM>
void launch_k3_team(gnna_ctx* ctx, AggArgs& a, uint32_t kmax, uint64_t grid, const gnna_plan* plan) {
    const bool fan = a.npeer || a.mc;
    constexpr bool kEW = std::is_same<T, float>::value;  // weighted gathers: fp32 path only
    if (fan && a.nw && (!kEW || kmax != 1))
        gnna::raise(GNNA_ERR_DOMAIN, "aggregate_fanout: node weights need fp32 rows of one chunk per lane");
    // split-node carries are combined by their last writer, zero-degree rows by
    // trailing blocks: one launch per aggregation
    a.unit_blocks = grid;
    a.nempty = plan->nempty;
    a.empty_rows = plan->fix_nodes.get() + plan->nsplit;
    a.carry_split = plan->carry_split.get();
    a.split_cnt = plan->split_cnt.get();
    a.split_node = plan->fix_nodes.get();
    a.split_first = plan->fix_first.get();
    a.split_count = plan->fix_count.get();
    if (k3a_applies<T, VEC, TEAM>(a, kmax)) {
        if constexpr (TEAM >= 2 && TEAM <= 8 && sizeof(T) * VEC == 16) {
            // 8 units per K3A CTA (64 threads for fp64 d 16): C3 fp64 0.093 ->
            // 0.088 ms (16: 0.089); GNNA_K3A_UPC=0 keeps K3's units per CTA
            static const int k3a_upc = [] {
                const char* e = std::getenv("GNNA_K3A_UPC");
                return e && *e ? std::atoi(e) : 8;
            }();
            if (k3a_upc > 0 && (uint32_t)k3a_upc < a.upc) {
                a.upc = std::max<uint32_t>(plan->wpb, ((uint32_t)k3a_upc / plan->wpb) * plan->wpb);
                grid = (plan->G + a.upc - 1) / a.upc;
                a.unit_blocks = grid;
            }
            const unsigned threads = (a.upc * TEAM + 31) / 32 * 32;
            const uint64_t total = grid + (a.nempty + threads / TEAM - 1) / (threads / TEAM);
            if (total > 0x7fffffffull) gnna::raise(GNNA_ERR_DOMAIN, "aggregate: grid too large");
            if (fan) launch_k3a_v<T, VEC, TEAM, false, true>(ctx, a, total, threads);
            else if (a.nw && kEW) launch_k3a_v<T, VEC, TEAM, kEW, false>(ctx, a, total, threads);
            else launch_k3a_v<T, VEC, TEAM, false, false>(ctx, a, total, threads);
        }
        return;
    }
    const size_t smem = (size_t)a.upc * kmax * TEAM * sizeof(Vec<T, VEC>);
    const unsigned threads = (a.upc * TEAM + 31) / 32 * 32;  // whole warps (gather_team is warp-collective)
    const uint64_t total = grid + (a.nempty + threads / TEAM - 1) / (threads / TEAM);
    if (!total) return;
    if (total > 0x7fffffffull) gnna::raise(GNNA_ERR_DOMAIN, "aggregate: grid too large");
    const unsigned g = (unsigned)total;
    if (fan && a.nw) {  // fused all-gather of a per-source-weighted gather (GCN's norm[u]), fp32
        k3_aggregate<T, VEC, TEAM, 1, kEW, true><<<g, threads, smem, ctx->stream>>>(a);
    } else if (fan) {  // fused all-gather: fp32 and fp64, unweighted gathers
        if (kmax == 1)
            k3_aggregate<T, VEC, TEAM, 1, false, true><<<g, threads, smem, ctx->stream>>>(a);
        else if (kmax == 2)
            k3_aggregate<T, VEC, TEAM, 2, false, true><<<g, threads, smem, ctx->stream>>>(a);
        else
            k3_aggregate<T, VEC, TEAM, 4, false, true><<<g, threads, smem, ctx->stream>>>(a);
    } else if (a.nw && kEW) {
        if (kmax == 1)
            k3_aggregate<T, VEC, TEAM, 1, kEW><<<g, threads, smem, ctx->stream>>>(a);
        else if (kmax == 2)
            k3_aggregate<T, VEC, TEAM, 2, kEW><<<g, threads, smem, ctx->stream>>>(a);
        else
            k3_aggregate<T, VEC, TEAM, 4, kEW><<<g, threads, smem, ctx->stream>>>(a);
    } else if (kmax == 1)
        k3_aggregate<T, VEC, TEAM, 1, false><<<g, threads, smem, ctx->stream>>>(a);
    else if (kmax == 2)
        k3_aggregate<T, VEC, TEAM, 2, false><<<g, threads, smem, ctx->stream>>>(a);
    else
        k3_aggregate<T, VEC, TEAM, 4, false><<<g, threads, smem, ctx->stream>>>(a);
    gnna::launched(ctx, "k3_aggregate");
    if ((kmax > 1 || TEAM > 8) && plan->nsplit) {
        const unsigned sg = (unsigned)((plan->nsplit + 256 / TEAM - 1) / (256 / TEAM));
        if (fan)
            k3b_split<T, VEC, TEAM, true><<<sg, 256, 0, ctx->stream>>>(a, plan->nsplit);
        else
            k3b_split<T, VEC, TEAM, false><<<sg, 256, 0, ctx->stream>>>(a, plan->nsplit);
        gnna::launched(ctx, "k3b_split");
    }
}

template <class T, int VEC>
void launch_k3(gnna_ctx* ctx, AggArgs& a, const Shape& s, uint64_t grid, const gnna_plan* plan) {
    switch (s.team) {
        case 1: launch_k3_team<T, VEC, 1>(ctx, a, s.kmax, grid, plan); break;
        case 2: launch_k3_team<T, VEC, 2>(ctx, a, s.kmax, grid, plan); break;
        case 4: launch_k3_team<T, VEC, 4>(ctx, a, s.kmax, grid, plan); break;
        case 8: launch_k3_team<T, VEC, 8>(ctx, a, s.kmax, grid, plan); break;
        case 16: launch_k3_team<T, VEC, 16>(ctx, a, s.kmax, grid, plan); break;
        default: launch_k3_team<T, VEC, 32>(ctx, a, s.kmax, grid, plan); break;
    }
}

template <class T, int VEC, int TEAM, int MODE>
void launch_k4_team(gnna_ctx* ctx, AggArgs& a, uint32_t kmax) {
    const unsigned grid = (unsigned)((a.units + 256 / TEAM - 1) / (256 / TEAM));
    if (kmax == 1)
        k4_rows<T, VEC, TEAM, 1, MODE><<<grid, 256, 0, ctx->stream>>>(a);
    else if (kmax == 2)
        k4_rows<T, VEC, TEAM, 2, MODE><<<grid, 256, 0, ctx->stream>>>(a);
    else
        k4_rows<T, VEC, TEAM, 4, MODE><<<grid, 256, 0, ctx->stream>>>(a);
    gnna::launched(ctx, "k4_rows");
}

template <class T, int VEC, int MODE>
void launch_k4(gnna_ctx* ctx, AggArgs& a, const Shape& s) {
    switch (s.team) {
        case 1: launch_k4_team<T, VEC, 1, MODE>(ctx, a, s.kmax); break;
        case 2: launch_k4_team<T, VEC, 2, MODE>(ctx, a, s.kmax); break;
        case 4: launch_k4_team<T, VEC, 4, MODE>(ctx, a, s.kmax); break;
        case 8: launch_k4_team<T, VEC, 8, MODE>(ctx, a, s.kmax); break;
        case 16: launch_k4_team<T, VEC, 16, MODE>(ctx, a, s.kmax); break;
        default: launch_k4_team<T, VEC, 32, MODE>(ctx, a, s.kmax); break;
    }
}

}  // namespace

// xs[u] = w[u] * x[u] for every row (the per-source weights of a weighted
// gather applied once per row instead of once per edge).
__global__ void k_prescale_rows(const float* __restrict__ x, const float* __restrict__ w, uint32_t n, uint32_t dim,
                                float* __restrict__ xs) {
    const uint64_t total = (uint64_t)n * dim;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    if (dim % 4 == 0 && (uintptr_t)x % 16 == 0 && (uintptr_t)xs % 16 == 0) {
        const uint32_t d4 = dim / 4;
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total / 4; i += stride) {
            const float c = __ldg(w + i / d4);
            const float4 v = __ldg(reinterpret_cast<const float4*>(x) + i);
            reinterpret_cast<float4*>(xs)[i] = make_float4(c * v.x, c * v.y, c * v.z, c * v.w);
        }
    } else {
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride)
            xs[i] = __ldg(w + i / dim) * __ldg(x + i);
    }
}

namespace gnna {

// Scheduled aggregation over a plan (one K3 / K3A launch) with the optional epilogue
// and per-edge weights of gnna_agg_opts (o may be null).
void aggregate_plan_fan(gnna_ctx* ctx, const gnna_plan* plan, int dtype, int dim_mode, const void* x, void* y,
                        const gnna_agg_opts* o, void* const* peers, uint32_t npeer, void* mc) {
    if (!plan) raise(GNNA_ERR_DOMAIN, "null plan");
    if (dtype != GNNA_F32 && dtype != GNNA_F64) raise(GNNA_ERR_DOMAIN, "unknown dtype");
    const uint32_t dim = (o && o->dim) ? o->dim : plan->params.dim;
    const int elem = dtype == GNNA_F32 ? 4 : 8;
    if (o && o->node_weight && dtype != GNNA_F32)
        raise(GNNA_ERR_DOMAIN, "aggregate: node weights are supported on the F32 path only");
    const uint32_t wpb = plan->wpb;
    bool others = !(o && o->mask) || (uintptr_t)o->mask % 16 == 0;
    for (uint32_t i = 0; i < npeer && peers; ++i) others = others && (uintptr_t)peers[i] % 16 == 0;
    others = others && (uintptr_t)mc % 16 == 0;
    const Shape s = choose_shape(elem, dim, plan->params.dw, pow2floor(256 / wpb), x, y, others);
    // carry slots are sized for the widest dim seen on this plan
    const uint64_t need = plan->ncarry * (uint64_t)dim * 8;
    if (need > plan->carry.n) {  // grow on the caller's stream, the old slots freed after their last use
        plan->carry.release_on(ctx->stream);
        plan->carry = DevBuf<uint8_t>(need, ctx->stream);
    }
    AggArgs a{};
    a.part_ptr = plan->part_ptr.get();
    a.part2node = plan->part2node.get();
    a.uflags = plan->uflags.get();
    a.cidx = plan->cidx.get();
    a.units = plan->G;
    a.upc = ((256 / s.team) / wpb) * wpb;
    {
        // at most 32 units per CTA: for narrow teams (d 16 fp32: 4 lanes) a
        // 256-thread CTA held 64 units and lived as long as the longest; 128
        // threads trim that tail (C3 sum 53.4 -> 52.7 us, train step 0.331 ->
        // 0.324 ms; C4 / C5 unchanged).  GNNA_K3_UPC_MAX=0 restores 256
        // threads, other values cap.
        static const int upc_max = [] {
            const char* e = std::getenv("GNNA_K3_UPC_MAX");
            return e && *e ? std::atoi(e) : 32;
        }();
        if (upc_max > 0) a.upc = std::min<uint32_t>(a.upc, std::max<uint32_t>(wpb, ((uint32_t)upc_max / wpb) * wpb));
    }
    a.row_ptr = plan->row_ptr;
    a.col = plan->col;
    a.x = x;
    a.y = y;
    a.carry = plan->carry.get();
    a.dim = dim;
    a.nvec = dim / s.vec;
    a.kpl = s.kpl;
    a.seq = dim_mode == GNNA_DIM_SEQUENTIAL;
    if (o) {
        if (o->self_weight || o->alpha != 0.0) a.epi |= EPI_SELF;
        if (o->row_scale) a.epi |= EPI_SCALE;
        if (o->relu) a.epi |= EPI_RELU;
        if (o->mask) a.epi |= EPI_MASK;
        a.sw = o->self_weight;
        a.alpha = o->alpha;
        a.scale = o->row_scale;
        a.mask = o->mask;
        a.nw = o->node_weight;
    }
    if (npeer > GNNA_MAX_PEERS) raise(GNNA_ERR_DOMAIN, "aggregate: at most GNNA_MAX_PEERS peer replicas");
    for (uint32_t i = 0; i < npeer; ++i) {
        if (!peers[i]) raise(GNNA_ERR_DOMAIN, "aggregate: null peer replica");
        a.peers[i] = peers[i];
    }
    a.npeer = npeer;
    a.mc = mc;
    {
        static const int pf_env = std::getenv("GNNA_K3_PF") ? std::atoi(std::getenv("GNNA_K3_PF")) : -1;
        a.pf = pf_env >= 0 ? (uint32_t)pf_env : (uint32_t)(3 * ctx->num_sms);  // ~ the resident CTAs of one wave
    }
    if (plan->G == 0 && plan->nempty == 0) return;
    // Per-source weights (GCN's norm[u] on an arbitrary x): with enough edges
    // per row, scale each row once into a scratch copy and gather that with
    // the plain K3 (the self term still reads the caller's x): C3 76.4 ->
    // 66.5 us, C5 15.7 -> 14.4 ms (profiles r02j).  Rounding: rn(w x) then the
    // sum, as in the GCN layer form, against fmaf per edge; the fused fan-out
    // takes the same path, so its replicas hold the same bits.
    // GNNA_PRESCALE=0 keeps the per-edge weights.
    DevBuf<float> xs;
    bool window_moved = false;
    cudaStreamAttrValue window_saved{};
    {
        static const int pre_env = std::getenv("GNNA_PRESCALE") ? std::atoi(std::getenv("GNNA_PRESCALE")) : -1;
        const uint32_t rows = plan->row_end - plan->row_begin;
        const bool pre = a.nw && dtype == GNNA_F32 &&
                         (pre_env >= 0 ? pre_env != 0 : plan->nnz >= 4ull * (rows ? rows : 1));
        if (pre) {
            xs = DevBuf<float>((size_t)plan->n * dim, ctx->stream);
            const uint64_t work = (uint64_t)plan->n * dim / (dim % 4 == 0 ? 4 : 1);
            const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, 16ull * ctx->num_sms));
            k_prescale_rows<<<blocks, 256, 0, ctx->stream>>>(static_cast<const float*>(x), a.nw, plan->n, dim, xs.get());
            launched(ctx, "k_prescale_rows");
            a.xself = x;
            a.x = xs.get();
            a.nw = nullptr;
            // an L2 persisting window the caller set on rows of x (gnna_set_l2_window) follows
            // the gather to the same rows of the scaled copy for this launch
            cudaStreamAttrValue w{};
            if (cudaStreamGetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &w) == cudaSuccess) {
                const auto* lo = static_cast<const unsigned char*>(x);
                const auto* bp = static_cast<const unsigned char*>(w.accessPolicyWindow.base_ptr);
                const size_t xbytes = (size_t)plan->n * dim * sizeof(float);
                if (w.accessPolicyWindow.num_bytes && bp >= lo && bp < lo + xbytes) {
                    window_saved = w;
                    cudaStreamAttrValue moved = w;
                    moved.accessPolicyWindow.base_ptr = reinterpret_cast<unsigned char*>(xs.get()) + (bp - lo);
                    moved.accessPolicyWindow.num_bytes = std::min<size_t>(w.accessPolicyWindow.num_bytes, xbytes - (bp - lo));
                    GNNA_CUDA(cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &moved));
                    window_moved = true;
                }
            } else {
                cudaGetLastError();
            }
        }
    }
    struct RestoreWindow {
        gnna_ctx* ctx;
        const bool& moved;
        cudaStreamAttrValue& saved;
        ~RestoreWindow() {
            if (moved) cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &saved);
        }
    } restore{ctx, window_moved, window_saved};
    const uint64_t grid = plan->G ? (plan->G + a.upc - 1) / a.upc : 0;  // unit blocks
    if (dtype == GNNA_F32) {
        if (s.vec == 4) launch_k3<float, 4>(ctx, a, s, grid, plan);
        else launch_k3<float, 1>(ctx, a, s, grid, plan);
    } else {
        if (s.vec == 2) launch_k3<double, 2>(ctx, a, s, grid, plan);
        else launch_k3<double, 1>(ctx, a, s, grid, plan);
    }
}

void aggregate_plan_ex(gnna_ctx* ctx, const gnna_plan* plan, int dtype, int dim_mode, const void* x, void* y,
                       const gnna_agg_opts* o) {
    aggregate_plan_fan(ctx, plan, dtype, dim_mode, x, y, o, nullptr, 0, nullptr);
}

void aggregate_plan(gnna_ctx* ctx, const gnna_plan* plan, int dtype, int dim_mode, const void* x, void* y,
                    uint32_t epi, const float* scale, double alpha) {
    gnna_agg_opts o{};
    o.row_scale = (epi & EPI_SCALE) ? scale : nullptr;
    o.alpha = (epi & EPI_SELF) ? alpha : 0.0;
    o.relu = (epi & EPI_RELU) ? 1 : 0;
    aggregate_plan_ex(ctx, plan, dtype, dim_mode, x, y, epi ? &o : nullptr);
}

// Row-order aggregation (K4).  mode 0 sum, 1 exact normalized, 2 exact GIN input.
void aggregate_rows(gnna_ctx* ctx, int dtype, const uint64_t* row_ptr, const uint32_t* col, uint32_t r0,
                    uint32_t rows, uint32_t dim, const void* x, void* y, int mode, const double* norm,
                    const uint8_t* self, double alpha, uint32_t epi, const float* scale) {
    if (dtype != GNNA_F32 && dtype != GNNA_F64) raise(GNNA_ERR_DOMAIN, "unknown dtype");
    if (rows == 0 || dim == 0) return;
    const int elem = dtype == GNNA_F32 ? 4 : 8;
    const Shape s = choose_shape(elem, dim, 32 * 4, 32, x, y);
    AggArgs a{};
    a.units = rows;
    a.r0 = r0;
    a.row_ptr = row_ptr;
    a.col = col;
    a.x = x;
    a.y = y;
    a.dim = dim;
    a.nvec = dim / s.vec;
    a.kpl = s.kpl;
    a.seq = 0;
    a.epi = epi;
    a.scale = scale;
    a.alpha = alpha;
    a.norm = norm;
    a.self = self;
    if (dtype == GNNA_F32) {
        if (mode == 1) {
            if (s.vec == 4) launch_k4<float, 4, 1>(ctx, a, s); else launch_k4<float, 1, 1>(ctx, a, s);
        } else if (mode == 2) {
            if (s.vec == 4) launch_k4<float, 4, 2>(ctx, a, s); else launch_k4<float, 1, 2>(ctx, a, s);
        } else {
            if (s.vec == 4) launch_k4<float, 4, 0>(ctx, a, s); else launch_k4<float, 1, 0>(ctx, a, s);
        }
    } else {
        if (mode == 1) {
            if (s.vec == 2) launch_k4<double, 2, 1>(ctx, a, s); else launch_k4<double, 1, 1>(ctx, a, s);
        } else if (mode == 2) {
            if (s.vec == 2) launch_k4<double, 2, 2>(ctx, a, s); else launch_k4<double, 1, 2>(ctx, a, s);
        } else {
            if (s.vec == 2) launch_k4<double, 2, 0>(ctx, a, s); else launch_k4<double, 1, 0>(ctx, a, s);
        }
    }
}

}  // namespace gnna

extern "C" {

gnna_status gnna_aggregate_ex(gnna_ctx* ctx, const gnna_plan* plan, int dtype, int dim_mode, const void* d_x,
                              void* d_y, const gnna_agg_opts* opts) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        gnna::aggregate_plan_ex(ctx, plan, dtype, dim_mode, d_x, d_y, opts);
    });
}

gnna_status gnna_aggregate_fanout(gnna_ctx* ctx, const gnna_plan* plan, int dtype, int dim_mode, const void* d_x,
                                  void* d_y, const gnna_agg_opts* opts, void* const* peer_y, uint32_t n_peer,
                                  void* mc_y) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (n_peer && !peer_y) gnna::raise(GNNA_ERR_DOMAIN, "aggregate_fanout: null peer list");
        gnna::aggregate_plan_fan(ctx, plan, dtype, dim_mode, d_x, d_y, opts, peer_y, n_peer, mc_y);
    });
}

gnna_status gnna_aggregate(gnna_ctx* ctx, const gnna_plan* plan, int dtype, int dim_mode, const void* d_x,
                           void* d_y) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        gnna::aggregate_plan(ctx, plan, dtype, dim_mode, d_x, d_y, 0, nullptr, 0.0);
    });
}

gnna_status gnna_aggregate_rows(gnna_ctx* ctx, int dtype, const uint64_t* d_row_ptr, const uint32_t* d_col,
                                uint32_t n, uint32_t dim, const void* d_x, void* d_y) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        gnna::aggregate_rows(ctx, dtype, d_row_ptr, d_col, 0, n, dim, d_x, d_y, 0, nullptr, nullptr, 0.0, 0,
                             nullptr);
    });
}

}  // extern "C"

extern "C" gnna_status gnna_tune_params(gnna_ctx* ctx, const uint64_t* d_row_ptr, const uint32_t* d_col, uint32_t n,
                                        uint32_t dim, const uint32_t* gs_values, uint32_t n_gs,
                                        const uint32_t* dw_values, uint32_t n_dw, const uint32_t* tpb_values,
                                        uint32_t n_tpb, gnna_params* best, float* best_ms) {
    // Measured-latency evaluator: the analytic model of
    // decider.cpp:70-81 replaced by CUDA-event timings of K3 on the live graph.
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (!best || !n_gs || !n_dw || !n_tpb) gnna::raise(GNNA_ERR_DOMAIN, "tune_params: empty grid");
        cudaStream_t s = ctx->stream;
        gnna::DevBuf<float> x((size_t)n * dim + 4, s), y((size_t)n * dim + 4, s);
        GNNA_CUDA(cudaMemsetAsync(x.get(), 0, ((size_t)n * dim + 4) * 4, s));
        cudaEvent_t e0, e1;
        GNNA_CUDA(cudaEventCreate(&e0));
        GNNA_CUDA(cudaEventCreate(&e1));
        float best_t = 3.4e38f;
        gnna_params bp{};
        bool found = false;
        for (uint32_t i = 0; i < n_gs; ++i)
            for (uint32_t j = 0; j < n_dw; ++j)
                for (uint32_t k = 0; k < n_tpb; ++k) {
                    gnna_params p{gs_values[i], dw_values[j], tpb_values[k], 32, dim};
                    gnna_plan* plan = nullptr;
                    if (gnna_plan_create(ctx, d_row_ptr, d_col, n, 0, n, &p, GNNA_WARP_SHARED, &plan) != GNNA_OK)
                        continue;  // infeasible combination (validate() domain)
                    gnna::aggregate_plan(ctx, plan, GNNA_F32, GNNA_DIM_CYCLIC, x.get(), y.get(), 0, nullptr, 0.0);
                    GNNA_CUDA(cudaEventRecord(e0, s));
                    const int reps = 3;
                    for (int r = 0; r < reps; ++r)
                        gnna::aggregate_plan(ctx, plan, GNNA_F32, GNNA_DIM_CYCLIC, x.get(), y.get(), 0, nullptr, 0.0);
                    GNNA_CUDA(cudaEventRecord(e1, s));
                    GNNA_CUDA(cudaEventSynchronize(e1));
                    float ms = 0;
                    GNNA_CUDA(cudaEventElapsedTime(&ms, e0, e1));
                    ms /= reps;
                    gnna_plan_destroy(plan);
                    if (ms < best_t) {
                        best_t = ms;
                        bp = p;
                        found = true;
                    }
                }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (!found) gnna::raise(GNNA_ERR_DOMAIN, "tune_params: no feasible combination");
        *best = bp;
        if (best_ms) *best_ms = best_t;
    });
}
