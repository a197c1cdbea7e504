// detect_communities on the GPU: the reference's exact greedy modularity
// agglomeration (renumber.cpp:31-104), merge for merge.
//
// Reference semantics reproduced bit for bit:
//   * m = number of unique undirected non-loop edges; every community pair
//     (a,b) with between-weight w has gain  w/m - (d_a*d_b)/((2m)m)  in IEEE
//     double with separately rounded operations (renumber.cpp:63);
//   * the merged pair is the maximum under the total order (gain desc, a asc,
//     b asc) over all live pairs (renumber.cpp:59-71); stop when that gain is
//     <= 0 (renumber.cpp:73);
//   * b merges into a = min(a,b): degrees add, between-maps union
//     (renumber.cpp:75-87); community names are their minimum member;
//   * dense ids follow ascending community name (= order of first appearance
//     by node id, renumber.cpp:91-101).
// Degrees and weights are integer counts held exactly (u64 / u32) and
// converted to double only inside the gain expression, as the reference's
// doubles hold exact integers.
//
// The merge ORDER is inherently sequential; the work of each merge is not.
// Layout and parallel decomposition:
//   * every live community owns an open-addressing hash table (neighbor ->
//     between-weight, one u64 slot = key<<32 | weight) in a slot pool;
//   * best[c] caches c's best pair under the total order (the survey's
//     cached-best restatement); after merging b into a only a's row and the
//     cache entries of a∪b's neighbours can change;
//   * a two-level max (blocks of 1024 communities) finds the global best pair.
// The merge loop is one persistent CTA of 1024 threads (state lives in L2);
// table construction and the initial caches are grid-wide kernels.  When the
// pool fills, live tables are compacted into a second pool (ping-pong).
#include <algorithm>

#include "gnna_common.cuh"

namespace gnna {
uint64_t undirected_edges(gnna_ctx* ctx, const uint64_t* row_ptr, const uint32_t* col, uint32_t n,
                          DevBuf<uint64_t>& out);
}

namespace {

using gnna::DevBuf;

constexpr uint32_t EMPTY = 0xffffffffu;
constexpr uint32_t TOMB = 0xfffffffeu;
constexpr uint32_t NONE = 0xffffffffu;
constexpr int CTA = 1024;
constexpr int BS = 1024;  // communities per max-block

struct Key {
    double g;
    uint32_t lo, hi;
};

__device__ __forceinline__ bool better(const Key& x, const Key& y) {
    if (x.g != y.g) return x.g > y.g;
    if (x.lo != y.lo) return x.lo < y.lo;
    return x.hi < y.hi;
}

__device__ __forceinline__ Key none_key() { return Key{-INFINITY, NONE, NONE}; }

struct State {
    uint32_t n;
    double m;
    double two_m_m;             // (2.0*m)*m
    unsigned long long* deg;    // [n]
    uint8_t* alive;             // [n]
    uint32_t* parent;           // [n] merge forest (b -> a)
    unsigned long long* pool[2];
    uint64_t pool_size;
    int cur;                    // current pool
    unsigned long long* top;    // [2] bump pointers
    uint64_t* off;              // [n] table offset in the current pool
    uint32_t* cap;              // [n] table capacity (power of 2)
    uint32_t* used;             // [n] slots taken (live + tombstones)
    uint32_t* live;             // [n] live entries
    double* bgain;              // [n] cached best pair of c
    uint32_t* bpart;            // [n]
    uint8_t* dirty;             // [nblk]
    Key* blk;                   // [nblk]
    uint32_t nblk;
    uint32_t* list;             // [n] scratch
    unsigned* err;              // 1 probe overflow, 2 pool exhausted
    unsigned long long* merges; // out
};

__device__ __forceinline__ double gain_of(const State& s, uint32_t w, uint64_t da, uint64_t db) {
    // renumber.cpp:63  w / m - deg_sum[a] * deg_sum[b] / (2.0 * m * m)
    return __dsub_rn(__ddiv_rn((double)w, s.m), __ddiv_rn(__dmul_rn((double)da, (double)db), s.two_m_m));
}

__device__ __forceinline__ uint32_t hslot(uint32_t key, uint32_t cap) {
    const int lg = __ffs(cap) - 1;
    return lg ? (uint32_t)(((uint64_t)key * 0x9E3779B97F4A7C15ull) >> (64 - lg)) : 0u;
}

__device__ __forceinline__ unsigned long long* table(const State& s, uint32_t c) { return s.pool[s.cur] + s.off[c]; }

// Add w to key in row (insert when absent).  Returns true if a new slot was
// taken.  Safe for concurrent adds into one row as long as it has room.
__device__ bool row_add(const State& s, unsigned long long* t, uint32_t cap, uint32_t key, uint32_t w) {
    uint32_t i = hslot(key, cap);
    for (uint32_t probe = 0; probe < cap; ++probe, i = (i + 1) & (cap - 1)) {
        unsigned long long v = *reinterpret_cast<volatile unsigned long long*>(t + i);
        for (;;) {
            const uint32_t k = (uint32_t)(v >> 32);
            if (k == key) {
                atomicAdd(t + i, (unsigned long long)w);
                return false;
            }
            if (k != EMPTY) break;
            const unsigned long long want = ((unsigned long long)key << 32) | w;
            const unsigned long long old = atomicCAS(t + i, v, want);
            if (old == v) return true;
            v = old;  // someone filled it: re-examine this slot
        }
    }
    atomicExch(s.err, 1u);
    return false;
}

__device__ bool row_erase(const State& s, unsigned long long* t, uint32_t cap, uint32_t key) {
    uint32_t i = hslot(key, cap);
    for (uint32_t probe = 0; probe < cap; ++probe, i = (i + 1) & (cap - 1)) {
        const unsigned long long v = t[i];
        const uint32_t k = (uint32_t)(v >> 32);
        if (k == key) {
            t[i] = (unsigned long long)TOMB << 32;
            return true;
        }
        if (k == EMPTY) return false;
    }
    return false;
}

__device__ __forceinline__ uint32_t pow2_at_least(uint32_t v) {
    uint32_t p = 4;
    while (p < v) p <<= 1;
    return p;
}

__device__ __forceinline__ bool slot_live(unsigned long long v) {
    const uint32_t k = (uint32_t)(v >> 32);
    return k != EMPTY && k != TOMB;
}

// ------------------------------------------------------------ setup kernels
__global__ void kc_degrees(const uint64_t* __restrict__ e, uint64_t m, unsigned long long* __restrict__ deg) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        atomicAdd(deg + (e[i] >> 32), 1ull);
        atomicAdd(deg + (uint32_t)e[i], 1ull);
    }
}

__global__ void kc_caps(const unsigned long long* __restrict__ deg, uint32_t n, uint32_t* __restrict__ cap,
                        uint64_t* __restrict__ capw) {
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < n; c += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t p = 4;
        while (p < 2 * deg[c]) p <<= 1;
        cap[c] = p;
        capw[c] = p;
    }
}

__global__ void kc_fill_empty(unsigned long long* __restrict__ p, uint64_t count) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = (unsigned long long)EMPTY << 32;
}

__global__ void kc_insert_edges(State s, const uint64_t* __restrict__ e, uint64_t m) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t a = (uint32_t)(e[i] >> 32), b = (uint32_t)e[i];
        row_add(s, table(s, a), s.cap[a], b, 1u);
        row_add(s, table(s, b), s.cap[b], a, 1u);
    }
}

__global__ void kc_init_rows(State s) {
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < s.n; c += (uint64_t)gridDim.x * blockDim.x) {
        s.alive[c] = 1;
        s.parent[c] = (uint32_t)c;
        s.used[c] = (uint32_t)s.deg[c];
        s.live[c] = (uint32_t)s.deg[c];
    }
}

// Best pair of row c (warp-cooperative).
__device__ Key warp_row_best(const State& s, uint32_t c, uint32_t lane) {
    Key best = none_key();
    const unsigned long long* t = table(s, c);
    const uint32_t cap = s.cap[c];
    const uint64_t dc = s.deg[c];
    for (uint32_t i = lane; i < cap; i += 32) {
        const unsigned long long v = t[i];
        if (!slot_live(v)) continue;
        const uint32_t d = (uint32_t)(v >> 32);
        const Key k{gain_of(s, (uint32_t)v, dc, s.deg[d]), min(c, d), max(c, d)};
        if (better(k, best)) best = k;
    }
    for (int o = 16; o; o >>= 1) {
        Key k{__shfl_xor_sync(0xffffffffu, best.g, o), __shfl_xor_sync(0xffffffffu, best.lo, o),
              __shfl_xor_sync(0xffffffffu, best.hi, o)};
        if (better(k, best)) best = k;
    }
    return best;
}

__device__ __forceinline__ void set_best(const State& s, uint32_t c, const Key& k) {
    s.bgain[c] = k.g;
    s.bpart[c] = k.lo == NONE ? NONE : (k.lo == c ? k.hi : k.lo);
}

__device__ __forceinline__ Key best_key(const State& s, uint32_t c) {
    const uint32_t p = s.bpart[c];
    if (!s.alive[c] || p == NONE) return none_key();
    return Key{s.bgain[c], min(c, p), max(c, p)};
}

__global__ void kc_init_best(State s) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t c = blockIdx.x * (uint64_t)(blockDim.x / 32) + threadIdx.x / 32; c < s.n; c += warps) {
        const Key k = warp_row_best(s, (uint32_t)c, lane);
        if (lane == 0) set_best(s, (uint32_t)c, k);
    }
}

// ------------------------------------------------------- CTA-wide helpers
__device__ Key cta_reduce(Key k, Key* sh) {
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x / 32;
    for (int o = 16; o; o >>= 1) {
        Key q{__shfl_xor_sync(0xffffffffu, k.g, o), __shfl_xor_sync(0xffffffffu, k.lo, o),
              __shfl_xor_sync(0xffffffffu, k.hi, o)};
        if (better(q, k)) k = q;
    }
    __syncthreads();
    if (lane == 0) sh[w] = k;
    __syncthreads();
    if (w == 0) {
        k = lane < blockDim.x / 32 ? sh[lane] : none_key();
        for (int o = 16; o; o >>= 1) {
            Key q{__shfl_xor_sync(0xffffffffu, k.g, o), __shfl_xor_sync(0xffffffffu, k.lo, o),
                  __shfl_xor_sync(0xffffffffu, k.hi, o)};
            if (better(q, k)) k = q;
        }
        if (lane == 0) sh[0] = k;
    }
    __syncthreads();
    const Key r = sh[0];
    __syncthreads();
    return r;
}

// ------------------------------------------------------------ merge loop
__global__ void __launch_bounds__(CTA) kc_merge_loop(State s) {
    __shared__ Key red[32];
    __shared__ uint32_t sh_a, sh_b, sh_nlist, sh_stop;
    __shared__ unsigned long long sh_off;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid / 32;
    // block maxima
    for (uint32_t k = warp; k < s.nblk; k += CTA / 32) {
        Key best = none_key();
        for (uint32_t c = k * BS + lane; c < min(s.n, (k + 1) * BS); c += 32) {
            const Key q = best_key(s, c);
            if (better(q, best)) best = q;
        }
        for (int o = 16; o; o >>= 1) {
            Key q{__shfl_xor_sync(0xffffffffu, best.g, o), __shfl_xor_sync(0xffffffffu, best.lo, o),
                  __shfl_xor_sync(0xffffffffu, best.hi, o)};
            if (better(q, best)) best = q;
        }
        if (lane == 0) {
            s.blk[k] = best;
            s.dirty[k] = 0;
        }
    }
    __syncthreads();
    unsigned long long merges = 0;
    for (uint32_t iter = 0; iter < s.n; ++iter) {
        // ---- global best pair
        Key best = none_key();
        for (uint32_t k = tid; k < s.nblk; k += CTA)
            if (better(s.blk[k], best)) best = s.blk[k];
        best = cta_reduce(best, red);
        if (best.lo == NONE || !(best.g > 0.0) || *s.err) break;  // renumber.cpp:73
        const uint32_t a = best.lo, b = best.hi;

        // ---- pool compaction when the next merge might not fit
        const uint64_t reserve = (uint64_t)32 * (uint64_t)s.m + 4096;
        if (s.top[s.cur] + reserve > s.pool_size) {
            const int dst = s.cur ^ 1;
            if (tid == 0) s.top[dst] = 0;
            __syncthreads();
            // one thread per live community: allocate + rehash sequentially
            for (uint32_t c = tid; c < s.n; c += CTA) {
                if (!s.alive[c]) continue;
                const uint32_t nc = pow2_at_least(2 * s.live[c] + 2);
                const unsigned long long o = atomicAdd(s.top + dst, (unsigned long long)nc);
                if (o + nc > s.pool_size) {
                    atomicExch(s.err, 2u);
                    continue;
                }
                unsigned long long* nt = s.pool[dst] + o;
                for (uint32_t i = 0; i < nc; ++i) nt[i] = (unsigned long long)EMPTY << 32;
                const unsigned long long* ot = s.pool[s.cur] + s.off[c];
                for (uint32_t i = 0; i < s.cap[c]; ++i)
                    if (slot_live(ot[i])) {
                        const uint32_t key = (uint32_t)(ot[i] >> 32);
                        uint32_t j = hslot(key, nc);
                        while ((uint32_t)(nt[j] >> 32) != EMPTY) j = (j + 1) & (nc - 1);
                        nt[j] = ot[i];
                    }
                s.off[c] = o;
                s.cap[c] = nc;
                s.used[c] = s.live[c];
            }
            __syncthreads();
            s.cur = dst;
            if (*s.err) break;
        }

        // ---- make room in row a for the union (rebuild if needed)
        if (s.used[a] + s.live[b] + 1 > s.cap[a] / 4 * 3) {
            const uint32_t nc = pow2_at_least(2 * (s.live[a] + s.live[b]) + 2);
            if (tid == 0) sh_off = atomicAdd(s.top + s.cur, (unsigned long long)nc);
            __syncthreads();
            const uint64_t o = sh_off;
            if (o + nc > s.pool_size) {
                if (tid == 0) atomicExch(s.err, 2u);
                break;
            }
            unsigned long long* nt = s.pool[s.cur] + o;
            for (uint32_t i = tid; i < nc; i += CTA) nt[i] = (unsigned long long)EMPTY << 32;
            __syncthreads();
            const unsigned long long* ot = table(s, a);
            for (uint32_t i = tid; i < s.cap[a]; i += CTA) {
                const unsigned long long v = ot[i];
                if (slot_live(v)) row_add(s, nt, nc, (uint32_t)(v >> 32), (uint32_t)v);
            }
            __syncthreads();
            if (tid == 0) {
                s.off[a] = o;
                s.cap[a] = nc;
                s.used[a] = s.live[a];
            }
            __syncthreads();
        }

        // ---- merge b into a (renumber.cpp:75-87)
        if (tid == 0) {
            s.deg[a] += s.deg[b];
            s.alive[b] = 0;
            s.parent[b] = a;
            if (row_erase(s, table(s, a), s.cap[a], b)) s.live[a] -= 1;
            sh_nlist = 0;
        }
        __syncthreads();
        {
            unsigned long long* ta = table(s, a);
            const uint32_t capa = s.cap[a];
            const unsigned long long* tb = table(s, b);
            for (uint32_t i = tid; i < s.cap[b]; i += CTA) {
                const unsigned long long v = tb[i];
                if (!slot_live(v)) continue;
                const uint32_t c = (uint32_t)(v >> 32), w = (uint32_t)v;
                if (c == a) continue;
                if (row_add(s, ta, capa, c, w)) {
                    atomicAdd(s.used + a, 1u);
                    atomicAdd(s.live + a, 1u);
                }
                // row c: erase b, add w to a (only this thread touches row c)
                unsigned long long* tc = table(s, c);
                row_erase(s, tc, s.cap[c], b);
                s.live[c] -= 1;
                if (s.used[c] + 1 > s.cap[c] / 4 * 3) {
                    const uint32_t nc = pow2_at_least(2 * (s.live[c] + 1) + 2);
                    const unsigned long long o = atomicAdd(s.top + s.cur, (unsigned long long)nc);
                    if (o + nc > s.pool_size) {
                        atomicExch(s.err, 2u);
                        continue;
                    }
                    unsigned long long* nt = s.pool[s.cur] + o;
                    for (uint32_t j = 0; j < nc; ++j) nt[j] = (unsigned long long)EMPTY << 32;
                    for (uint32_t j = 0; j < s.cap[c]; ++j)
                        if (slot_live(tc[j])) {
                            const uint32_t key = (uint32_t)(tc[j] >> 32);
                            uint32_t q = hslot(key, nc);
                            while ((uint32_t)(nt[q] >> 32) != EMPTY) q = (q + 1) & (nc - 1);
                            nt[q] = tc[j];
                        }
                    s.off[c] = o;
                    s.cap[c] = nc;
                    s.used[c] = s.live[c];
                    tc = nt;
                }
                if (row_add(s, tc, s.cap[c], a, w)) {
                    s.used[c] += 1;
                    s.live[c] += 1;
                }
            }
        }
        __syncthreads();
        // ---- caches: best[a] in full; neighbours of a∪b
        {
            const unsigned long long* ta = table(s, a);
            const uint32_t capa = s.cap[a];
            const uint64_t da = s.deg[a];
            Key ka = none_key();
            for (uint32_t i = tid; i < capa; i += CTA) {
                const unsigned long long v = ta[i];
                if (!slot_live(v)) continue;
                const uint32_t c = (uint32_t)(v >> 32);
                const uint64_t dc = s.deg[c];
                const Key k{gain_of(s, (uint32_t)v, da, dc), min(a, c), max(a, c)};
                if (better(k, ka)) ka = k;
                // neighbour c's cache
                const uint32_t p = s.bpart[c];
                if (p == a || p == b) {
                    s.list[atomicAdd(&sh_nlist, 1u)] = c;
                } else {
                    const Key kc{gain_of(s, (uint32_t)v, dc, da), min(a, c), max(a, c)};
                    const Key cur = p == NONE ? none_key() : Key{s.bgain[c], min(c, p), max(c, p)};
                    if (better(kc, cur)) set_best(s, c, kc);
                }
                s.dirty[c / BS] = 1;
            }
            ka = cta_reduce(ka, red);
            if (tid == 0) {
                set_best(s, a, ka);
                s.bpart[b] = NONE;
                s.dirty[a / BS] = 1;
                s.dirty[b / BS] = 1;
            }
        }
        __syncthreads();
        for (uint32_t j = warp; j < sh_nlist; j += CTA / 32) {
            const uint32_t c = s.list[j];
            const Key k = warp_row_best(s, c, lane);
            if (lane == 0) set_best(s, c, k);
        }
        __syncthreads();
        // ---- refresh dirty block maxima
        for (uint32_t k = warp; k < s.nblk; k += CTA / 32) {
            if (!s.dirty[k]) continue;
            Key bk = none_key();
            for (uint32_t c = k * BS + lane; c < min(s.n, (k + 1) * BS); c += 32) {
                const Key q = best_key(s, c);
                if (better(q, bk)) bk = q;
            }
            for (int o = 16; o; o >>= 1) {
                Key q{__shfl_xor_sync(0xffffffffu, bk.g, o), __shfl_xor_sync(0xffffffffu, bk.lo, o),
                      __shfl_xor_sync(0xffffffffu, bk.hi, o)};
                if (better(q, bk)) bk = q;
            }
            if (lane == 0) {
                s.blk[k] = bk;
                s.dirty[k] = 0;
            }
        }
        __syncthreads();
        ++merges;
    }
    if (tid == 0) *s.merges = merges;
    (void)sh_a;
    (void)sh_b;
    (void)sh_stop;
}

// --------------------------------------------------------------- labels
__global__ void kc_roots(const uint32_t* __restrict__ parent, uint32_t n, uint32_t* __restrict__ root,
                         uint32_t* __restrict__ is_root) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t r = (uint32_t)v;
        while (parent[r] != r) r = parent[r];
        root[v] = r;
        is_root[v] = r == v ? 1u : 0u;
    }
}

__global__ void kc_labels(const uint32_t* __restrict__ root, const uint64_t* __restrict__ rank, uint32_t n,
                          uint32_t* __restrict__ com) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x)
        com[v] = (uint32_t)rank[root[v]];
}

}  // namespace

extern "C" gnna_status gnna_detect_communities(gnna_ctx* ctx, const uint64_t* d_row_ptr, const uint32_t* d_col,
                                               uint32_t n, uint32_t* d_com, uint32_t* num_communities) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        cudaStream_t st = ctx->stream;
        if (n == 0) {
            *num_communities = 0;
            return;
        }
        DevBuf<uint64_t> e;
        const uint64_t m = gnna::undirected_edges(ctx, d_row_ptr, d_col, n, e);
        DevBuf<unsigned long long> deg(n, st);
        GNNA_CUDA(cudaMemsetAsync(deg.get(), 0, (size_t)n * 8, st));
        if (m) {
            kc_degrees<<<gnna::grid_for(m, 256), 256, 0, st>>>(e.get(), m, deg.get());
            gnna::launched(ctx, "kc_degrees");
        }
        DevBuf<uint32_t> cap(n, st), used(n, st), live(n, st), parent(n, st), bpart(n, st), list(n, st);
        DevBuf<uint64_t> capw(n, st), off((uint64_t)n + 1, st);
        DevBuf<uint8_t> alive(n, st);
        DevBuf<double> bgain(n, st);
        kc_caps<<<gnna::grid_for(n, 256), 256, 0, st>>>(deg.get(), n, cap.get(), capw.get());
        gnna::launched(ctx, "kc_caps");
        const uint64_t init_slots = gnna::exclusive_scan_u64(ctx, capw.get(), off.get(), n);
        const uint64_t pool_size = std::max<uint64_t>(init_slots, 8 * m + 8 * (uint64_t)n) + 40 * m + 65536;
        DevBuf<unsigned long long> pool0(pool_size, st), pool1(m ? pool_size : 1, st), top(2, st);
        kc_fill_empty<<<gnna::grid_for(init_slots, 256), 256, 0, st>>>(pool0.get(), init_slots);
        gnna::launched(ctx, "kc_fill_empty");
        const unsigned long long tops[2] = {init_slots, 0};
        GNNA_CUDA(cudaMemcpyAsync(top.get(), tops, sizeof(tops), cudaMemcpyHostToDevice, st));
        const uint32_t nblk = (n + BS - 1) / BS;
        DevBuf<uint8_t> dirty(nblk, st);
        DevBuf<Key> blk(nblk, st);
        DevBuf<unsigned> err(1, st);
        DevBuf<unsigned long long> merges(1, st);
        GNNA_CUDA(cudaMemsetAsync(err.get(), 0, 4, st));
        GNNA_CUDA(cudaMemsetAsync(merges.get(), 0, 8, st));
        State s{};
        s.n = n;
        s.m = (double)m;
        s.two_m_m = (2.0 * s.m) * s.m;
        s.deg = deg.get();
        s.alive = alive.get();
        s.parent = parent.get();
        s.pool[0] = pool0.get();
        s.pool[1] = pool1.get();
        s.pool_size = pool_size;
        s.cur = 0;
        s.top = top.get();
        s.off = off.get();
        s.cap = cap.get();
        s.used = used.get();
        s.live = live.get();
        s.bgain = bgain.get();
        s.bpart = bpart.get();
        s.dirty = dirty.get();
        s.blk = blk.get();
        s.nblk = nblk;
        s.list = list.get();
        s.err = err.get();
        s.merges = merges.get();
        kc_init_rows<<<gnna::grid_for(n, 256), 256, 0, st>>>(s);
        gnna::launched(ctx, "kc_init_rows");
        if (m) {
            kc_insert_edges<<<gnna::grid_for(m, 256), 256, 0, st>>>(s, e.get(), m);
            gnna::launched(ctx, "kc_insert_edges");
            kc_init_best<<<gnna::grid_for((uint64_t)n * 32, 256), 256, 0, st>>>(s);
            gnna::launched(ctx, "kc_init_best");
            kc_merge_loop<<<1, CTA, 0, st>>>(s);
            gnna::launched(ctx, "kc_merge_loop");
            unsigned h = 0;
            gnna::to_host(ctx, &h, err.get(), 1);
            if (h == 1) gnna::raise(GNNA_ERR_INTERNAL, "detect_communities: hash table overflow");
            if (h == 2) gnna::raise(GNNA_ERR_OOM, "detect_communities: adjacency pool exhausted");
        }
        DevBuf<uint32_t> root(n, st), isroot(n, st);
        DevBuf<uint64_t> rank((uint64_t)n + 1, st);
        kc_roots<<<gnna::grid_for(n, 256), 256, 0, st>>>(parent.get(), n, root.get(), isroot.get());
        gnna::launched(ctx, "kc_roots");
        const uint64_t k = gnna::exclusive_scan_u32_to_u64(ctx, isroot.get(), rank.get(), n);
        kc_labels<<<gnna::grid_for(n, 256), 256, 0, st>>>(root.get(), rank.get(), n, d_com);
        gnna::launched(ctx, "kc_labels");
        GNNA_CUDA(cudaStreamSynchronize(st));
        *num_communities = (uint32_t)k;
    });
}
