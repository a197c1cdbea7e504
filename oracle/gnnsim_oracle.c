/* TEST INFRASTRUCTURE ONLY — CPU parity oracle for the gnnsim aggregation
 * path.  See gnnsim_oracle.h for the contract.  Each function cites the
 * reference file:line (under /root/reference/proj) it restates.  Plain C11,
 * compiled -O2 without -march (no FMA contraction; -std=c11 also turns off
 * -ffp-contract), matching the reference build's floating-point behaviour.
 */
#include "gnnsim_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* orc_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- RNG --- */
/* std::mt19937_64 (the reference's engine) + rand.hpp:13-21 draws. */
#define MT_N 312
#define MT_M 156
void orc_rng_seed(orc_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = MT_N;
}

uint64_t orc_rng_next(orc_rng* r) {
    if (r->idx >= MT_N) {
        for (int i = 0; i < MT_N; ++i) {
            uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) |
                         (r->mt[(i + 1) % MT_N] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* rand.hpp:13 draw_index: 128-bit multiply-shift. */
uint64_t orc_draw_index(orc_rng* r, uint64_t n) {
    return (uint64_t)(((unsigned __int128)orc_rng_next(r) * n) >> 64);
}

/* rand.hpp:19 draw_unit: 53 random bits. */
double orc_draw_unit(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }

/* pipeline.cpp:57-67 random_features */
int orc_random_features(uint32_t n, uint32_t dim, uint64_t seed, double* out) {
    if (dim == 0) return fail(1, "dim must be positive");
    orc_rng r;
    orc_rng_seed(&r, seed);
    for (uint64_t i = 0; i < (uint64_t)n * dim; ++i) out[i] = orc_draw_unit(&r);
    return 0;
}

/* pipeline.cpp:14-48 planted_partition */
int orc_planted_partition(uint32_t communities, uint32_t size, double p_in, double p_out,
                          int shuffle, uint64_t seed, uint64_t cap, uint32_t* edges,
                          uint64_t* num_edges, uint32_t* num_nodes) {
    if (communities == 0 || size == 0)
        return fail(1, "need at least one community of at least one node");
    if (!(p_in >= 0.0 && p_in <= 1.0) || !(p_out >= 0.0 && p_out <= 1.0))
        return fail(1, "edge probabilities must lie in [0, 1]");
    uint64_t total = (uint64_t)communities * size;
    if (total > (1u << 16)) return fail(1, "generator samples all node pairs; limit is 65536 nodes");
    uint32_t n = (uint32_t)total;
    orc_rng r;
    orc_rng_seed(&r, seed);
    uint64_t e = 0;
    for (uint32_t i = 0; i < n; ++i) {
        uint32_t ci = i / size;
        for (uint32_t j = i + 1; j < n; ++j) {
            double p = (j / size == ci) ? p_in : p_out;
            if (orc_draw_unit(&r) < p) {
                if (e < cap) {
                    edges[2 * e] = i;
                    edges[2 * e + 1] = j;
                }
                ++e;
            }
        }
    }
    *num_edges = e;
    *num_nodes = n;
    if (e > cap) return fail(6, "caller buffer too small");
    if (shuffle) {
        uint32_t* perm = malloc(sizeof(uint32_t) * (n ? n : 1));
        for (uint32_t i = 0; i < n; ++i) perm[i] = i;
        for (uint32_t i = n; i > 1; --i) {
            uint64_t j = orc_draw_index(&r, i);
            uint32_t t = perm[i - 1];
            perm[i - 1] = perm[j];
            perm[j] = t;
        }
        for (uint64_t k = 0; k < 2 * e; ++k) edges[k] = perm[edges[k]];
        free(perm);
    }
    return 0;
}

/* -------------------------------------------------------------- graph --- */
static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : x > y;
}
static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : x > y;
}

/* graph.cpp:76-95 to_csr: bucket per row (both directions when symmetrizing),
 * sort each row ascending, drop duplicates. */
int orc_to_csr(uint32_t n, const uint32_t* edges, uint64_t e, int symmetrize,
               uint64_t* row_ptr, uint32_t* col, uint64_t col_cap, uint64_t* nnz) {
    uint64_t* cnt = calloc((size_t)n + 1, sizeof(uint64_t));
    for (uint64_t i = 0; i < e; ++i) {
        if (edges[2 * i] >= n || edges[2 * i + 1] >= n) {
            free(cnt);
            return fail(1, "edge endpoint out of range");
        }
        cnt[edges[2 * i] + 1]++;
        if (symmetrize) cnt[edges[2 * i + 1] + 1]++;
    }
    for (uint32_t v = 0; v < n; ++v) cnt[v + 1] += cnt[v];
    uint64_t total = cnt[n];
    uint32_t* tmp = malloc(sizeof(uint32_t) * (total ? total : 1));
    uint64_t* fill = malloc(sizeof(uint64_t) * ((size_t)n + 1));
    memcpy(fill, cnt, sizeof(uint64_t) * ((size_t)n + 1));
    for (uint64_t i = 0; i < e; ++i) {
        uint32_t u = edges[2 * i], v = edges[2 * i + 1];
        tmp[fill[u]++] = v;
        if (symmetrize) tmp[fill[v]++] = u;
    }
    uint64_t out = 0;
    row_ptr[0] = 0;
    int rc = 0;
    for (uint32_t v = 0; v < n; ++v) {
        uint32_t* row = tmp + cnt[v];
        uint64_t len = cnt[v + 1] - cnt[v];
        qsort(row, len, sizeof(uint32_t), cmp_u32);
        for (uint64_t k = 0; k < len; ++k) {
            if (k > 0 && row[k] == row[k - 1]) continue;
            if (out < col_cap) col[out] = row[k];
            ++out;
        }
        row_ptr[v + 1] = out;
    }
    *nnz = out;
    if (out > col_cap) rc = fail(6, "caller buffer too small");
    free(cnt);
    free(tmp);
    free(fill);
    return rc;
}

/* graph.cpp:122-128 aes: double running sum of |src - dst| / E. */
int orc_aes(uint32_t n, const uint32_t* edges, uint64_t e, double* out) {
    (void)n;
    if (e == 0) return fail(1, "no edges in the input");
    double s = 0.0;
    for (uint64_t i = 0; i < e; ++i) {
        uint32_t u = edges[2 * i], v = edges[2 * i + 1];
        s += (double)(u > v ? u - v : v - u);
    }
    *out = s / (double)e;
    return 0;
}

/* renumber.cpp:198-201 should_reorder */
int orc_should_reorder(uint32_t n, const uint32_t* edges, uint64_t e, int* out) {
    double a;
    int rc = orc_aes(n, edges, e, &a);
    if (rc) return rc;
    double threshold = floor(sqrt((double)n) / 100.0);
    *out = sqrt(a) > threshold;
    return 0;
}

/* graph.cpp:106-120 degree_stats */
int orc_degree_stats(uint32_t n, const uint64_t* row_ptr, const uint32_t* col, double* avg,
                     uint64_t* maxd, double* sd) {
    (void)col;
    if (n == 0) return fail(1, "degree_stats: graph has no nodes");
    double dn = (double)n;
    double a = (double)row_ptr[n] / dn;
    double sq = 0.0;
    uint64_t mx = 0;
    for (uint32_t v = 0; v < n; ++v) {
        uint64_t d = row_ptr[v + 1] - row_ptr[v];
        if (d > mx) mx = d;
        double dc = (double)d - a;
        sq += dc * dc;
    }
    *avg = a;
    *maxd = mx;
    *sd = sqrt(sq / dn);
    return 0;
}

/* ----------------------------------------------------------- schedule --- */
/* schedule.cpp:7-14 KernelParams::validate (same order, same messages).
 * p = {ngs, dw, tpb, tpw, dim}. */
int orc_validate_params(const uint32_t p[5]) {
    if (p[0] < 1) return fail(1, "params: ngs must be >= 1");
    if (p[3] != 32) return fail(1, "params: tpw is fixed at 32");
    if (p[1] < 1 || p[1] > p[3]) return fail(1, "params: dw must be in [1, tpw]");
    if (p[2] == 0 || p[2] % p[3] != 0) return fail(1, "params: tpb must be a positive multiple of tpw");
    if (p[2] > 1024) return fail(1, "params: tpb must be <= 1024");
    if (p[4] < 1) return fail(1, "params: dim must be >= 1");
    return 0;
}

/* schedule.cpp:16-30 partition_neighbors */
int orc_partition_neighbors(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                            uint32_t ngs, uint64_t cap, uint64_t* num_groups, uint32_t* ids,
                            uint32_t* targets, uint64_t* begins, uint64_t* ends) {
    (void)col;
    if (ngs < 1) return fail(1, "partition_neighbors: ngs must be >= 1");
    uint64_t g = 0;
    for (uint32_t v = 0; v < n; ++v) {
        uint64_t b = row_ptr[v], re = row_ptr[v + 1];
        while (b < re) {
            uint64_t e = b + ngs < re ? b + ngs : re;
            if (g < cap) {
                ids[g] = (uint32_t)g;
                targets[g] = v;
                begins[g] = b;
                ends[g] = e;
            }
            ++g;
            b = e;
        }
    }
    *num_groups = g;
    return g > cap ? fail(6, "caller buffer too small") : 0;
}

/* schedule.cpp:32-47 partition_dims: lanes flattened as lane_ptr[dw+1]. */
int orc_partition_dims(uint32_t dim, uint32_t dw, int mode, uint32_t* lane_ptr,
                       uint32_t* dims) {
    if (dw < 1) return fail(1, "partition_dims: dw must be >= 1");
    uint32_t k = 0;
    lane_ptr[0] = 0;
    if (mode == 0) {
        uint32_t chunk = (dim + dw - 1) / dw;
        for (uint32_t t = 0; t < dw; ++t) {
            uint32_t hi = (t + 1) * chunk < dim ? (t + 1) * chunk : dim;
            for (uint32_t d = t * chunk; d < hi; ++d) dims[k++] = d;
            lane_ptr[t + 1] = k;
        }
    } else {
        for (uint32_t t = 0; t < dw; ++t) {
            for (uint32_t d = t; d < dim; d += dw) dims[k++] = d;
            lane_ptr[t + 1] = k;
        }
    }
    return 0;
}

/* memplan.cpp:9-63 build_mem_plan (Algorithm 1), including the
 * consecutive-run precondition (memplan.cpp:15-29). */
int orc_build_mem_plan(const uint32_t* targets, uint64_t num_groups, const uint32_t p[5],
                       uint32_t* slots, uint32_t* nodes, uint8_t* leaders,
                       uint64_t* smem_bytes) {
    int rc = orc_validate_params(p);
    if (rc) return rc;
    uint32_t wpb = p[2] / p[3];
    /* consecutive check: a target may not reappear after its run closed */
    if (num_groups > 0) {
        uint32_t maxt = 0;
        for (uint64_t i = 0; i < num_groups; ++i)
            if (targets[i] > maxt) maxt = targets[i];
        uint8_t* closed = calloc((size_t)maxt + 1, 1);
        for (uint64_t i = 0; i < num_groups; ++i) {
            if (i > 0 && targets[i] == targets[i - 1]) continue;
            if (closed[targets[i]]) {
                free(closed);
                snprintf(g_err, sizeof g_err, "build_mem_plan: warps of node %u are not consecutive",
                         targets[i]);
                return 1;
            }
            if (i > 0) closed[targets[i - 1]] = 1;
        }
        free(closed);
    }
    *smem_bytes = (uint64_t)wpb * p[4] * 4;
    uint32_t local = 0, last = 0;
    for (uint64_t cnt = 0; cnt < num_groups;) {
        uint32_t node = targets[cnt];
        nodes[cnt] = node;
        if (cnt % wpb == 0) {
            slots[cnt] = local;
            last = node;
            leaders[cnt] = 1;
        } else if (node == last) {
            slots[cnt] = local;
            leaders[cnt] = 0;
        } else {
            ++local;
            slots[cnt] = local;
            last = node;
            leaders[cnt] = 1;
        }
        ++cnt;
        if (cnt % wpb == 0) local = 0;
    }
    return 0;
}

/* ------------------------------------------------------------- engine --- */
/* engine.cpp:36-49 step_lines over a flattened DimAssignment. */
static uint64_t step_lines(uint64_t base, const uint32_t* lane_ptr, const uint32_t* dims,
                           uint32_t dw, uint64_t iter, uint64_t line) {
    uint64_t cnt = 0, prev = UINT64_MAX;
    for (uint32_t t = 0; t < dw; ++t) {
        uint64_t len = lane_ptr[t + 1] - lane_ptr[t];
        if (iter >= len) continue;
        uint64_t l = (base + (uint64_t)dims[lane_ptr[t] + iter] * 4) / line;
        if (l != prev) {
            ++cnt;
            prev = l;
        }
    }
    return cnt;
}

/* LRU over 128-bit-free line ids: open addressing (linear probing,
 * backward-shift delete) + intrusive doubly-linked recency list.
 * Restates LruCache (engine.cpp:51-74). */
typedef struct {
    uint64_t* keys;
    int64_t* slot; /* hash -> node index, -1 empty */
    uint64_t mask;
    uint64_t* line; /* node -> line */
    int64_t *prev, *next;
    int64_t head, tail, free_head;
    uint64_t size, cap;
} lru_t;

static uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static void lru_init(lru_t* c, uint64_t cap, uint64_t max_distinct) {
    uint64_t need = (cap + 1 < max_distinct + 1 ? cap + 1 : max_distinct + 1);
    uint64_t sz = 4;
    while (sz < 2 * need) sz <<= 1;
    c->mask = sz - 1;
    c->keys = malloc(sizeof(uint64_t) * sz);
    c->slot = malloc(sizeof(int64_t) * sz);
    for (uint64_t i = 0; i < sz; ++i) c->slot[i] = -1;
    c->line = malloc(sizeof(uint64_t) * (need + 1));
    c->prev = malloc(sizeof(int64_t) * (need + 1));
    c->next = malloc(sizeof(int64_t) * (need + 1));
    for (uint64_t i = 0; i <= need; ++i) c->next[i] = (int64_t)i + 1 <= (int64_t)need ? (int64_t)i + 1 : -1;
    c->free_head = 0;
    c->head = c->tail = -1;
    c->size = 0;
    c->cap = cap;
}

static void lru_free(lru_t* c) {
    free(c->keys);
    free(c->slot);
    free(c->line);
    free(c->prev);
    free(c->next);
}

static int64_t lru_find(lru_t* c, uint64_t key, uint64_t* pos) {
    uint64_t h = mix64(key) & c->mask;
    while (c->slot[h] >= 0) {
        if (c->keys[h] == key) {
            *pos = h;
            return c->slot[h];
        }
        h = (h + 1) & c->mask;
    }
    *pos = h;
    return -1;
}

static void lru_hash_erase(lru_t* c, uint64_t key) {
    uint64_t h;
    if (lru_find(c, key, &h) < 0) return;
    c->slot[h] = -1;
    uint64_t j = h;
    for (;;) {
        j = (j + 1) & c->mask;
        if (c->slot[j] < 0) break;
        uint64_t home = mix64(c->keys[j]) & c->mask;
        /* move j back to h if home is not cyclically in (h, j] */
        int move = (h <= j) ? (home <= h || home > j) : (home <= h && home > j);
        if (move) {
            c->keys[h] = c->keys[j];
            c->slot[h] = c->slot[j];
            c->slot[j] = -1;
            h = j;
        }
    }
}

static void lru_unlink(lru_t* c, int64_t i) {
    if (c->prev[i] >= 0) c->next[c->prev[i]] = c->next[i]; else c->head = c->next[i];
    if (c->next[i] >= 0) c->prev[c->next[i]] = c->prev[i]; else c->tail = c->prev[i];
}

static void lru_push_front(lru_t* c, int64_t i) {
    c->prev[i] = -1;
    c->next[i] = c->head;
    if (c->head >= 0) c->prev[c->head] = i;
    c->head = i;
    if (c->tail < 0) c->tail = i;
}

/* engine.cpp:55-69 LruCache::touch */
static int lru_touch(lru_t* c, uint64_t line) {
    uint64_t pos;
    int64_t i = lru_find(c, line, &pos);
    if (i >= 0) {
        lru_unlink(c, i);
        lru_push_front(c, i);
        return 1;
    }
    i = c->free_head;
    c->free_head = c->next[i];
    c->line[i] = line;
    c->keys[pos] = line;
    c->slot[pos] = i;
    lru_push_front(c, i);
    c->size++;
    if (c->size > c->cap) {
        int64_t t = c->tail;
        lru_unlink(c, t);
        lru_hash_erase(c, c->line[t]);
        c->next[t] = c->free_head;
        c->free_head = t;
        c->size--;
    }
    return 0;
}

/* engine.cpp:78-101 replay_block_cache for groups [lo, hi). */
static void replay_block(const uint32_t* col, const uint64_t* begins, const uint64_t* ends,
                         uint64_t lo, uint64_t hi, uint64_t cap_bytes, uint64_t line_size,
                         uint32_t dim, uint64_t* hits, uint64_t* accesses) {
    uint64_t row_bytes = (uint64_t)dim * 4;
    uint64_t total = 0;
    for (uint64_t w = lo; w < hi; ++w)
        total += (ends[w] - begins[w]) * ((row_bytes + line_size - 1) / line_size + 1);
    lru_t c;
    lru_init(&c, cap_bytes / line_size, total);
    for (uint64_t k = 0;; ++k) {
        int any = 0;
        for (uint64_t w = lo; w < hi; ++w) {
            if (k >= ends[w] - begins[w]) continue;
            any = 1;
            uint64_t base = (uint64_t)col[begins[w] + k] * dim * 4;
            uint64_t first = base / line_size, last = (base + row_bytes - 1) / line_size;
            for (uint64_t l = first; l <= last; ++l) {
                ++*accesses;
                if (lru_touch(&c, l)) ++*hits;
            }
        }
        if (!any) break;
    }
    lru_free(&c);
}

static int cache_validate(uint64_t cap, uint64_t line) {
    /* engine.cpp:141-145 CacheConfig::validate */
    if (line == 0) return fail(1, "cache line size must be positive");
    if (cap < line || cap % line != 0)
        return fail(1, "cache capacity must be a positive multiple of the line size");
    return 0;
}

/* engine.cpp:149-160 aggregate_oracle */
int orc_aggregate_oracle(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                         const double* x, uint32_t dim, double* y) {
    memset(y, 0, sizeof(double) * n * (size_t)dim);
    for (uint32_t v = 0; v < n; ++v) {
        double* out = y + (size_t)v * dim;
        for (uint64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {
            const double* in = x + (size_t)col[e] * dim;
            for (uint32_t d = 0; d < dim; ++d) out[d] += in[d];
        }
    }
    return 0;
}

/* engine.cpp:174-183 count_transactions */
int orc_count_transactions(const uint64_t* addr, uint64_t k, uint64_t line, uint64_t* out) {
    if (line == 0) return fail(1, "transaction line size must be positive");
    uint64_t* l = malloc(sizeof(uint64_t) * (k ? k : 1));
    for (uint64_t i = 0; i < k; ++i) l[i] = addr[i] / line;
    qsort(l, k, sizeof(uint64_t), cmp_u64);
    uint64_t u = 0;
    for (uint64_t i = 0; i < k; ++i)
        if (i == 0 || l[i] != l[i - 1]) ++u;
    free(l);
    *out = u;
    return 0;
}

/* engine.cpp:185-198 simulate_cache */
int orc_simulate_cache(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                       const uint32_t p[5], uint64_t cache_cap, uint64_t cache_line,
                       uint32_t dim, uint64_t* hits, uint64_t* accesses) {
    int rc = cache_validate(cache_cap, cache_line);
    if (rc) return rc;
    if (dim == 0) return fail(1, "dim must be positive");
    rc = orc_validate_params(p);
    if (rc) return rc;
    uint64_t G = 0;
    for (uint32_t v = 0; v < n; ++v) G += (row_ptr[v + 1] - row_ptr[v] + p[0] - 1) / p[0];
    uint32_t* ids = malloc(sizeof(uint32_t) * (G ? G : 1));
    uint32_t* tg = malloc(sizeof(uint32_t) * (G ? G : 1));
    uint64_t* bg = malloc(sizeof(uint64_t) * (G ? G : 1));
    uint64_t* en = malloc(sizeof(uint64_t) * (G ? G : 1));
    orc_partition_neighbors(n, row_ptr, col, p[0], G, &G, ids, tg, bg, en);
    uint32_t wpb = p[2] / p[3];
    *hits = *accesses = 0;
    for (uint64_t lo = 0; lo < G; lo += wpb) {
        uint64_t hi = lo + wpb < G ? lo + wpb : G;
        replay_block(col, bg, en, lo, hi, cache_cap, cache_line, dim, hits, accesses);
    }
    free(ids);
    free(tg);
    free(bg);
    free(en);
    return 0;
}

/* engine.cpp:200-311 aggregate_scheduled.  Summation tree restated exactly:
 * per group a sequential partial in CSR order; WarpShared slots accumulate
 * partials in warp order and leaders flush in warp order; the serial merge
 * adds flushes block by block (which is what applying each block's flushes
 * in order, block after block, does).  `workers` cannot change the result
 * (engine.hpp:68-70) and is ignored. */
int orc_aggregate_scheduled(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                            const double* x, const uint32_t p[5], int strategy, int dim_mode,
                            uint32_t workers, uint64_t line, int cache_on, uint64_t cache_cap,
                            uint64_t cache_line, double* y, uint64_t cost[7]) {
    (void)workers;
    int rc = orc_validate_params(p);
    if (rc) return rc;
    const uint32_t ngs = p[0], dw = p[1], dim = p[4], wpb = p[2] / p[3];
    if (line == 0) return fail(1, "transaction line size must be positive");
    if (cache_on && (rc = cache_validate(cache_cap, cache_line))) return rc;

    uint64_t G = 0;
    for (uint32_t v = 0; v < n; ++v) G += (row_ptr[v + 1] - row_ptr[v] + ngs - 1) / ngs;
    size_t gsz = G ? G : 1;
    uint32_t* ids = malloc(sizeof(uint32_t) * gsz);
    uint32_t* tg = malloc(sizeof(uint32_t) * gsz);
    uint64_t* bg = malloc(sizeof(uint64_t) * gsz);
    uint64_t* en = malloc(sizeof(uint64_t) * gsz);
    orc_partition_neighbors(n, row_ptr, col, ngs, G, &G, ids, tg, bg, en);

    uint32_t* lane_ptr = malloc(sizeof(uint32_t) * (dw + 1));
    uint32_t* dims = malloc(sizeof(uint32_t) * (dim ? dim : 1));
    orc_partition_dims(dim, dw, dim_mode, lane_ptr, dims);
    const uint64_t iters = (dim + dw - 1) / dw;

    uint32_t* slots = NULL;
    uint32_t* nodes = NULL;
    uint8_t* leaders = NULL;
    uint64_t smem = 0;
    if (strategy == 2) {
        slots = malloc(sizeof(uint32_t) * gsz);
        nodes = malloc(sizeof(uint32_t) * gsz);
        leaders = malloc(gsz);
        rc = orc_build_mem_plan(tg, G, p, slots, nodes, leaders, &smem);
        if (rc) goto done;
    }

    memset(y, 0, sizeof(double) * n * (size_t)dim);
    memset(cost, 0, sizeof(uint64_t) * 7);
    double* partial = malloc(sizeof(double) * dim);
    double* slotbuf = malloc(sizeof(double) * (size_t)wpb * dim);
    for (uint64_t lo = 0; lo < G; lo += wpb) {
        uint64_t hi = lo + wpb < G ? lo + wpb : G;
        if (strategy == 2) memset(slotbuf, 0, sizeof(double) * (size_t)wpb * dim);
        for (uint64_t w = lo; w < hi; ++w) {
            uint64_t size = en[w] - bg[w];
            for (uint32_t d = 0; d < dim; ++d) partial[d] = 0.0;
            for (uint64_t q = bg[w]; q < en[w]; ++q) {
                uint32_t u = col[q];
                const double* in = x + (size_t)u * dim;
                for (uint32_t d = 0; d < dim; ++d) partial[d] += in[d];
                uint64_t base = (uint64_t)u * dim * 4;
                for (uint64_t i = 0; i < iters; ++i)
                    cost[3] += step_lines(base, lane_ptr, dims, dw, i, line);
                if (strategy == 0) {
                    uint64_t tb = (uint64_t)tg[w] * dim * 4;
                    for (uint64_t i = 0; i < iters; ++i)
                        cost[3] += step_lines(tb, lane_ptr, dims, dw, i, line);
                }
            }
            cost[1] += size * dim;
            if (strategy == 0) {
                cost[0] += size * dim;
                cost[2] += size * dim;
                double* row = y + (size_t)tg[w] * dim;
                for (uint32_t d = 0; d < dim; ++d) row[d] += partial[d];
            } else if (strategy == 1) {
                cost[0] += dim;
                cost[2] += dim;
                uint64_t tb = (uint64_t)tg[w] * dim * 4;
                for (uint64_t i = 0; i < iters; ++i)
                    cost[3] += step_lines(tb, lane_ptr, dims, dw, i, line);
                double* row = y + (size_t)tg[w] * dim;
                for (uint32_t d = 0; d < dim; ++d) row[d] += partial[d];
            } else {
                double* s = slotbuf + (size_t)slots[w] * dim;
                for (uint32_t d = 0; d < dim; ++d) s[d] += partial[d];
            }
        }
        if (strategy == 2) {
            for (uint64_t w = lo; w < hi; ++w) {
                if (!leaders[w]) continue;
                cost[0] += dim;
                cost[2] += dim;
                uint64_t tb = (uint64_t)nodes[w] * dim * 4;
                for (uint64_t i = 0; i < iters; ++i)
                    cost[3] += step_lines(tb, lane_ptr, dims, dw, i, line);
                double* row = y + (size_t)nodes[w] * dim;
                const double* s = slotbuf + (size_t)slots[w] * dim;
                for (uint32_t d = 0; d < dim; ++d) row[d] += s[d];
            }
        }
        if (cache_on) replay_block(col, bg, en, lo, hi, cache_cap, cache_line, dim, &cost[5], &cost[6]);
    }
    if (strategy == 2) cost[4] = smem;
    free(partial);
    free(slotbuf);
done:
    free(ids);
    free(tg);
    free(bg);
    free(en);
    free(lane_ptr);
    free(dims);
    free(slots);
    free(nodes);
    free(leaders);
    return rc;
}

/* ------------------------------------------------------------- layers --- */
/* engine.cpp:315-331 matmul: k ascending, zero a[i][k] skipped. */
static void matmul(const double* a, uint32_t rows, uint32_t k_dim, const double* w,
                   uint32_t cols, double* out) {
    memset(out, 0, sizeof(double) * rows * (size_t)cols);
    for (uint32_t i = 0; i < rows; ++i) {
        const double* ai = a + (size_t)i * k_dim;
        double* oi = out + (size_t)i * cols;
        for (uint32_t k = 0; k < k_dim; ++k) {
            double aik = ai[k];
            if (aik == 0.0) continue;
            const double* wk = w + (size_t)k * cols;
            for (uint32_t j = 0; j < cols; ++j) oi[j] += aik * wk[j];
        }
    }
}

static int row_has(const uint64_t* row_ptr, const uint32_t* col, uint32_t v, uint32_t u) {
    uint64_t lo = row_ptr[v], hi = row_ptr[v + 1];
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (col[mid] < u) lo = mid + 1; else hi = mid;
    }
    return lo < row_ptr[v + 1] && col[lo] == u;
}

/* engine.cpp:340-353 normalization: norm[v] = 1/sqrt(max(deg',1)). */
static void gcn_norm(uint32_t n, const uint64_t* row_ptr, const uint32_t* col, int self_loops,
                     double* norm, uint8_t* implicit_self) {
    for (uint32_t v = 0; v < n; ++v) {
        uint64_t deg = row_ptr[v + 1] - row_ptr[v];
        implicit_self[v] = 0;
        if (self_loops && !row_has(row_ptr, col, v, v)) {
            implicit_self[v] = 1;
            ++deg;
        }
        if (deg == 0) deg = 1;
        norm[v] = 1.0 / sqrt((double)deg);
    }
}

/* engine.cpp:338-369 normalized_aggregate */
static void normalized_aggregate(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                                 const double* x, uint32_t dim, const double* norm,
                                 const uint8_t* implicit_self, double* z) {
    memset(z, 0, sizeof(double) * n * (size_t)dim);
    for (uint32_t v = 0; v < n; ++v) {
        double* out = z + (size_t)v * dim;
        for (uint64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {
            uint32_t u = col[e];
            double c = norm[v] * norm[u];
            const double* in = x + (size_t)u * dim;
            for (uint32_t d = 0; d < dim; ++d) out[d] += c * in[d];
        }
        if (implicit_self[v]) {
            double c = norm[v] * norm[v];
            const double* in = x + (size_t)v * dim;
            for (uint32_t d = 0; d < dim; ++d) out[d] += c * in[d];
        }
    }
}

/* Transposed normalized aggregation: out[u] += norm[v]norm[u] g[v] for u in
 * N(v) (no reference; the adjoint of normalized_aggregate). */
static void normalized_aggregate_t(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                                   const double* g, uint32_t dim, const double* norm,
                                   const uint8_t* implicit_self, double* out) {
    memset(out, 0, sizeof(double) * n * (size_t)dim);
    for (uint32_t v = 0; v < n; ++v) {
        const double* gv = g + (size_t)v * dim;
        for (uint64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {
            uint32_t u = col[e];
            double c = norm[v] * norm[u];
            double* o = out + (size_t)u * dim;
            for (uint32_t d = 0; d < dim; ++d) o[d] += c * gv[d];
        }
        if (implicit_self[v]) {
            double c = norm[v] * norm[v];
            double* o = out + (size_t)v * dim;
            for (uint32_t d = 0; d < dim; ++d) o[d] += c * gv[d];
        }
    }
}

/* engine.cpp:373-382 gcn_layer */
int orc_gcn_layer(uint32_t n, const uint64_t* row_ptr, const uint32_t* col, const double* x,
                  uint32_t in_dim, const double* w, uint32_t out_dim, int self_loops,
                  double* y) {
    double* norm = malloc(sizeof(double) * (n ? n : 1));
    uint8_t* imp = malloc(n ? n : 1);
    gcn_norm(n, row_ptr, col, self_loops, norm, imp);
    if (out_dim < in_dim) {
        double* h = malloc(sizeof(double) * ((size_t)n * out_dim + 1));
        matmul(x, n, in_dim, w, out_dim, h);
        normalized_aggregate(n, row_ptr, col, h, out_dim, norm, imp, y);
        free(h);
    } else {
        double* z = malloc(sizeof(double) * ((size_t)n * in_dim + 1));
        normalized_aggregate(n, row_ptr, col, x, in_dim, norm, imp, z);
        matmul(z, n, in_dim, w, out_dim, y);
        free(z);
    }
    free(norm);
    free(imp);
    return 0;
}

/* a^T b for row-major a (rows x ka), b (rows x kb) -> out (ka x kb). */
static void matmul_tn(const double* a, uint32_t rows, uint32_t ka, const double* b, uint32_t kb,
                      double* out) {
    memset(out, 0, sizeof(double) * ka * (size_t)kb);
    for (uint32_t i = 0; i < rows; ++i)
        for (uint32_t p = 0; p < ka; ++p) {
            double av = a[(size_t)i * ka + p];
            for (uint32_t q = 0; q < kb; ++q) out[(size_t)p * kb + q] += av * b[(size_t)i * kb + q];
        }
}

/* a w^T for a (rows x kw_cols), w (k x kw_cols) -> out (rows x k). */
static void matmul_nt(const double* a, uint32_t rows, uint32_t cols, const double* w, uint32_t k,
                      double* out) {
    for (uint32_t i = 0; i < rows; ++i)
        for (uint32_t p = 0; p < k; ++p) {
            double s = 0.0;
            for (uint32_t q = 0; q < cols; ++q) s += a[(size_t)i * cols + q] * w[(size_t)p * cols + q];
            out[(size_t)i * k + p] = s;
        }
}

int orc_gcn_backward(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                     const double* x, uint32_t in_dim, const double* w, uint32_t out_dim,
                     int self_loops, const double* dy, double* dx, double* dw) {
    double* norm = malloc(sizeof(double) * (n ? n : 1));
    uint8_t* imp = malloc(n ? n : 1);
    gcn_norm(n, row_ptr, col, self_loops, norm, imp);
    if (out_dim < in_dim) {
        /* y = A (x w): dh = A^T dy; dw = x^T dh; dx = dh w^T */
        double* dh = malloc(sizeof(double) * ((size_t)n * out_dim + 1));
        normalized_aggregate_t(n, row_ptr, col, dy, out_dim, norm, imp, dh);
        matmul_tn(x, n, in_dim, dh, out_dim, dw);
        matmul_nt(dh, n, out_dim, w, in_dim, dx);
        free(dh);
    } else {
        /* y = (A x) w: dz = dy w^T; dw = z^T dy; dx = A^T dz */
        double* z = malloc(sizeof(double) * ((size_t)n * in_dim + 1));
        double* dz = malloc(sizeof(double) * ((size_t)n * in_dim + 1));
        normalized_aggregate(n, row_ptr, col, x, in_dim, norm, imp, z);
        matmul_tn(z, n, in_dim, dy, out_dim, dw);
        matmul_nt(dy, n, out_dim, w, in_dim, dz);
        normalized_aggregate_t(n, row_ptr, col, dz, in_dim, norm, imp, dx);
        free(z);
        free(dz);
    }
    free(norm);
    free(imp);
    return 0;
}

/* engine.cpp:384-408 gin_layer */
int orc_gin_layer(uint32_t n, const uint64_t* row_ptr, const uint32_t* col, const double* x,
                  uint32_t in_dim, double eps, const double* w, uint32_t out_dim,
                  const double* b, double* y) {
    double* z = malloc(sizeof(double) * ((size_t)n * in_dim + 1));
    orc_aggregate_oracle(n, row_ptr, col, x, in_dim, z);
    double scale = 1.0 + eps;
    for (size_t i = 0; i < (size_t)n * in_dim; ++i) z[i] += scale * x[i];
    matmul(z, n, in_dim, w, out_dim, y);
    for (uint32_t i = 0; i < n; ++i)
        for (uint32_t j = 0; j < out_dim; ++j) {
            double v = y[(size_t)i * out_dim + j] + b[j];
            y[(size_t)i * out_dim + j] = v > 0.0 ? v : 0.0; /* std::max(0.0, v) */
        }
    free(z);
    return 0;
}

int orc_gin_backward(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                     const double* x, uint32_t in_dim, double eps, const double* w,
                     uint32_t out_dim, const double* b, const double* dy, double* dx,
                     double* dw, double* db, double* deps) {
    size_t nz = (size_t)n * in_dim + 1, nu = (size_t)n * out_dim + 1;
    double* z = malloc(sizeof(double) * nz);
    double* u = malloc(sizeof(double) * nu);
    double* du = calloc(nu, sizeof(double));
    double* dz = malloc(sizeof(double) * nz);
    orc_aggregate_oracle(n, row_ptr, col, x, in_dim, z);
    double scale = 1.0 + eps;
    for (size_t i = 0; i < (size_t)n * in_dim; ++i) z[i] += scale * x[i];
    matmul(z, n, in_dim, w, out_dim, u);
    for (uint32_t j = 0; j < out_dim; ++j) db[j] = 0.0;
    for (uint32_t i = 0; i < n; ++i)
        for (uint32_t j = 0; j < out_dim; ++j) {
            size_t k = (size_t)i * out_dim + j;
            du[k] = (u[k] + b[j] > 0.0) ? dy[k] : 0.0;
            db[j] += du[k];
        }
    matmul_tn(z, n, in_dim, du, out_dim, dw);
    matmul_nt(du, n, out_dim, w, in_dim, dz);
    /* dx = A^T dz + (1+eps) dz;  deps = sum x . dz */
    memset(dx, 0, sizeof(double) * n * (size_t)in_dim);
    for (uint32_t v = 0; v < n; ++v)
        for (uint64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {
            double* o = dx + (size_t)col[e] * in_dim;
            const double* g = dz + (size_t)v * in_dim;
            for (uint32_t d = 0; d < in_dim; ++d) o[d] += g[d];
        }
    double de = 0.0;
    for (size_t i = 0; i < (size_t)n * in_dim; ++i) {
        dx[i] += scale * dz[i];
        de += x[i] * dz[i];
    }
    *deps = de;
    free(z);
    free(u);
    free(du);
    free(dz);
    return 0;
}

/* ---------------------------------------------------------- renumber --- */
/* renumber.cpp:16-27 undirected_edges: {min,max} keys, sorted, unique. */
static uint64_t undirected_edges(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                                 uint64_t** out) {
    uint64_t* k = malloc(sizeof(uint64_t) * (row_ptr[n] ? row_ptr[n] : 1));
    uint64_t m = 0;
    for (uint32_t v = 0; v < n; ++v)
        for (uint64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {
            uint32_t u = col[e];
            if (u == v) continue;
            uint32_t a = u < v ? u : v, b = u < v ? v : u;
            k[m++] = ((uint64_t)a << 32) | b;
        }
    qsort(k, m, sizeof(uint64_t), cmp_u64);
    uint64_t w = 0;
    for (uint64_t i = 0; i < m; ++i)
        if (i == 0 || k[i] != k[i - 1]) k[w++] = k[i];
    *out = k;
    return w;
}

/* Pair-weight map keyed by (min << 32 | max); grows by rehash. */
typedef struct {
    uint64_t* keys;
    double* vals;
    uint64_t mask, size;
} pmap;

static void pm_init(pmap* m, uint64_t expect) {
    uint64_t sz = 16;
    while (sz < 2 * expect) sz <<= 1;
    m->mask = sz - 1;
    m->size = 0;
    m->keys = malloc(sizeof(uint64_t) * sz);
    m->vals = malloc(sizeof(double) * sz);
    for (uint64_t i = 0; i < sz; ++i) m->keys[i] = UINT64_MAX;
}

static double* pm_slot(pmap* m, uint64_t key, int create);

static void pm_grow(pmap* m) {
    uint64_t old = m->mask + 1;
    uint64_t* ok = m->keys;
    double* ov = m->vals;
    pm_init(m, old);  /* doubles capacity: sz >= 2*old */
    for (uint64_t i = 0; i < old; ++i)
        if (ok[i] != UINT64_MAX) *pm_slot(m, ok[i], 1) = ov[i];
    free(ok);
    free(ov);
}

static double* pm_slot(pmap* m, uint64_t key, int create) {
    uint64_t h = mix64(key) & m->mask;
    while (m->keys[h] != UINT64_MAX) {
        if (m->keys[h] == key) return &m->vals[h];
        h = (h + 1) & m->mask;
    }
    if (!create) return NULL;
    if (2 * (m->size + 1) > m->mask + 1) {
        pm_grow(m);
        return pm_slot(m, key, 1);
    }
    m->keys[h] = key;
    m->vals[h] = 0.0;
    m->size++;
    return &m->vals[h];
}

static uint64_t pkey(uint32_t a, uint32_t b) {
    return a < b ? ((uint64_t)a << 32) | b : ((uint64_t)b << 32) | a;
}

typedef struct {
    uint32_t* v;
    uint64_t len, cap;
} u32vec;

static void vpush(u32vec* a, uint32_t x) {
    if (a->len == a->cap) {
        a->cap = a->cap ? 2 * a->cap : 4;
        a->v = realloc(a->v, sizeof(uint32_t) * a->cap);
    }
    a->v[a->len++] = x;
}

typedef struct {
    double gain;
    uint32_t a, b; /* pair, a < b */
    uint32_t owner;
    uint64_t ver;
} heap_ent;

/* total order of renumber.cpp:64-66: larger gain first, then smaller (a,b) */
static int ent_better(double g1, uint32_t a1, uint32_t b1, double g2, uint32_t a2, uint32_t b2) {
    if (g1 != g2) return g1 > g2;
    if (a1 != a2) return a1 < a2;
    return b1 < b2;
}

typedef struct {
    heap_ent* e;
    uint64_t len, cap;
} heap_t;

static void heap_push(heap_t* h, heap_ent x) {
    if (h->len == h->cap) {
        h->cap = h->cap ? 2 * h->cap : 64;
        h->e = realloc(h->e, sizeof(heap_ent) * h->cap);
    }
    uint64_t i = h->len++;
    while (i > 0) {
        uint64_t p = (i - 1) / 2;
        if (!ent_better(x.gain, x.a, x.b, h->e[p].gain, h->e[p].a, h->e[p].b)) break;
        h->e[i] = h->e[p];
        i = p;
    }
    h->e[i] = x;
}

static heap_ent heap_pop(heap_t* h) {
    heap_ent top = h->e[0];
    heap_ent x = h->e[--h->len];
    if (h->len == 0) return top;
    uint64_t i = 0;
    for (;;) {
        uint64_t l = 2 * i + 1, r = l + 1, c;
        if (l >= h->len) break;
        c = l;
        if (r < h->len && ent_better(h->e[r].gain, h->e[r].a, h->e[r].b, h->e[l].gain,
                                     h->e[l].a, h->e[l].b))
            c = r;
        if (!ent_better(h->e[c].gain, h->e[c].a, h->e[c].b, x.gain, x.a, x.b)) break;
        h->e[i] = h->e[c];
        i = c;
    }
    h->e[i] = x;
    return top;
}

/* renumber.cpp:63 gain, evaluated in the same operation order. */
static double cnm_gain(double w, double da, double db, double m) {
    return w / m - da * db / (2.0 * m * m);
}

/* renumber.cpp:31-104 detect_communities.  Same merge sequence as the
 * reference's full rescans, found faster: each community caches its best
 * partner under the reference's total order (gain desc, (a,b) asc) and a
 * lazy max-heap holds the cached bests.  After b merges into a, only pairs
 * touching a change; a neighbour c re-scans its row only when its cached
 * partner was a or b, otherwise it compares against the new (c,a) key.
 * Gains come from the same exact-integer doubles and expression, so each
 * arg-max equals the reference's. */
int orc_detect_communities(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                           uint32_t* com, uint32_t* ncom) {
    uint64_t* ue;
    uint64_t me = undirected_edges(n, row_ptr, col, &ue);
    double m = (double)me;
    double* deg = calloc(n ? n : 1, sizeof(double));
    uint8_t* alive = malloc(n ? n : 1);
    uint32_t* parent = malloc(sizeof(uint32_t) * (n ? n : 1));
    u32vec* adj = calloc(n ? n : 1, sizeof(u32vec));
    uint32_t* best_d = malloc(sizeof(uint32_t) * (n ? n : 1));
    double* best_g = malloc(sizeof(double) * (n ? n : 1));
    uint64_t* ver = calloc(n ? n : 1, sizeof(uint64_t));
    pmap pm;
    pm_init(&pm, me + 16);
    for (uint32_t v = 0; v < n; ++v) {
        alive[v] = 1;
        parent[v] = v;
        best_d[v] = UINT32_MAX;
    }
    for (uint64_t i = 0; i < me; ++i) {
        uint32_t u = (uint32_t)(ue[i] >> 32), v = (uint32_t)ue[i];
        deg[u] += 1.0;
        deg[v] += 1.0;
        *pm_slot(&pm, ue[i], 1) += 1.0;
        vpush(&adj[u], v);
        vpush(&adj[v], u);
    }
    free(ue);

    heap_t heap = {0};
    /* (re)scan c's row: compacts dead entries, recomputes best partner */
    #define RESCAN(c)                                                              \
        do {                                                                       \
            uint32_t _c = (c);                                                     \
            u32vec* _r = &adj[_c];                                                 \
            uint64_t _w = 0;                                                       \
            best_d[_c] = UINT32_MAX;                                               \
            for (uint64_t _i = 0; _i < _r->len; ++_i) {                            \
                uint32_t _d = _r->v[_i];                                           \
                if (!alive[_d] || _d == _c) continue;                              \
                _r->v[_w++] = _d;                                                  \
                double _g = cnm_gain(*pm_slot(&pm, pkey(_c, _d), 0), deg[_c], deg[_d], m); \
                uint32_t _a = _c < _d ? _c : _d, _b = _c < _d ? _d : _c;           \
                if (best_d[_c] == UINT32_MAX) {                                    \
                    best_d[_c] = _d; best_g[_c] = _g;                              \
                } else {                                                           \
                    uint32_t _pa = _c < best_d[_c] ? _c : best_d[_c];              \
                    uint32_t _pb = _c < best_d[_c] ? best_d[_c] : _c;              \
                    if (ent_better(_g, _a, _b, best_g[_c], _pa, _pb)) {            \
                        best_d[_c] = _d; best_g[_c] = _g;                          \
                    }                                                              \
                }                                                                  \
            }                                                                      \
            _r->len = _w;                                                          \
        } while (0)
    #define PUSH(c)                                                                \
        do {                                                                       \
            uint32_t _c = (c);                                                     \
            ver[_c]++;                                                             \
            if (best_d[_c] != UINT32_MAX) {                                        \
                heap_ent _e;                                                       \
                _e.gain = best_g[_c];                                              \
                _e.a = _c < best_d[_c] ? _c : best_d[_c];                          \
                _e.b = _c < best_d[_c] ? best_d[_c] : _c;                          \
                _e.owner = _c;                                                     \
                _e.ver = ver[_c];                                                  \
                heap_push(&heap, _e);                                              \
            }                                                                      \
        } while (0)

    if (me > 0) {
        for (uint32_t c = 0; c < n; ++c) {
            RESCAN(c);
            PUSH(c);
        }
        while (heap.len) {
            heap_ent top = heap_pop(&heap);
            if (!alive[top.owner] || top.ver != ver[top.owner]) continue;
            if (!(top.gain > 0.0)) break;
            uint32_t a = top.a, b = top.b; /* b merges into a */
            deg[a] += deg[b];
            for (uint64_t i = 0; i < adj[b].len; ++i) {
                uint32_t c = adj[b].v[i];
                if (!alive[c] || c == a || c == b) continue;
                double w = *pm_slot(&pm, pkey(b, c), 0);
                double* s = pm_slot(&pm, pkey(a, c), 0);
                if (s) {
                    *s += w;
                } else {
                    *pm_slot(&pm, pkey(a, c), 1) = w;
                    vpush(&adj[a], c);
                    vpush(&adj[c], a);
                }
            }
            alive[b] = 0;
            parent[b] = a;
            free(adj[b].v);
            adj[b].v = NULL;
            adj[b].len = adj[b].cap = 0;
            RESCAN(a);
            PUSH(a);
            for (uint64_t i = 0; i < adj[a].len; ++i) {
                uint32_t c = adj[a].v[i];
                if (best_d[c] == a || best_d[c] == b || best_d[c] == UINT32_MAX) {
                    RESCAN(c);
                } else {
                    double g = cnm_gain(*pm_slot(&pm, pkey(a, c), 0), deg[a], deg[c], m);
                    uint32_t pa = c < best_d[c] ? c : best_d[c], pb = c < best_d[c] ? best_d[c] : c;
                    uint32_t qa = a < c ? a : c, qb = a < c ? c : a;
                    if (!ent_better(g, qa, qb, best_g[c], pa, pb)) continue;
                    best_d[c] = a;
                    best_g[c] = g;
                }
                PUSH(c);
            }
        }
    }
    #undef RESCAN
    #undef PUSH

    /* renumber.cpp:91-101: dense ids by first appearance of each name. */
    uint32_t* dense = malloc(sizeof(uint32_t) * (n ? n : 1));
    for (uint32_t v = 0; v < n; ++v) dense[v] = UINT32_MAX;
    uint32_t next = 0;
    for (uint32_t v = 0; v < n; ++v) {
        uint32_t r = v;
        while (parent[r] != r) r = parent[r];
        if (dense[r] == UINT32_MAX) dense[r] = next++;
        com[v] = dense[r];
    }
    *ncom = next;
    for (uint32_t v = 0; v < n; ++v) free(adj[v].v);
    free(adj);
    free(dense);
    free(deg);
    free(alive);
    free(parent);
    free(best_d);
    free(best_g);
    free(ver);
    free(heap.e);
    free(pm.keys);
    free(pm.vals);
    return 0;
}

/* renumber.cpp:106-126 modularity */
int orc_modularity(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                   const uint32_t* com, uint32_t ncom, double* q) {
    uint64_t* ue;
    uint64_t me = undirected_edges(n, row_ptr, col, &ue);
    if (me == 0) {
        free(ue);
        *q = 0.0;
        return 0;
    }
    double m = (double)me;
    double* intra = calloc(ncom ? ncom : 1, sizeof(double));
    double* dg = calloc(ncom ? ncom : 1, sizeof(double));
    for (uint64_t i = 0; i < me; ++i) {
        uint32_t u = (uint32_t)(ue[i] >> 32), v = (uint32_t)ue[i];
        dg[com[u]] += 1.0;
        dg[com[v]] += 1.0;
        if (com[u] == com[v]) intra[com[u]] += 1.0;
    }
    double s = 0.0;
    for (uint32_t c = 0; c < ncom; ++c) {
        double frac = dg[c] / (2.0 * m);
        s += intra[c] / m - frac * frac;
    }
    *q = s;
    free(ue);
    free(intra);
    free(dg);
    return 0;
}

/* renumber.cpp:128-146 build_mapping: order by (community, old id). */
int orc_build_mapping(uint32_t n, const uint32_t* com, uint32_t ncom, uint32_t* o2n,
                      uint32_t* n2o) {
    uint64_t* start = calloc((size_t)ncom + 1, sizeof(uint64_t));
    for (uint32_t v = 0; v < n; ++v) {
        if (com[v] >= ncom) {
            free(start);
            return fail(1, "community id out of range");
        }
        start[com[v] + 1]++;
    }
    for (uint32_t c = 0; c < ncom; ++c) start[c + 1] += start[c];
    for (uint32_t v = 0; v < n; ++v) {
        uint32_t nv = (uint32_t)start[com[v]]++;
        o2n[v] = nv;
        n2o[nv] = v;
    }
    free(start);
    return 0;
}

/* renumber.cpp:148-160 mapping_from_vector */
int orc_mapping_from_vector(uint32_t n, const uint32_t* v, uint32_t* o2n, uint32_t* n2o) {
    for (uint32_t i = 0; i < n; ++i) n2o[i] = n;
    for (uint32_t i = 0; i < n; ++i) {
        uint32_t w = v[i];
        o2n[i] = w;
        if (w >= n || n2o[w] != n) return fail(1, "mapping is not a permutation of its index range");
        n2o[w] = i;
    }
    return 0;
}

/* renumber.cpp:162-185 apply_mapping (CSR) */
int orc_apply_mapping_csr(uint32_t n, const uint64_t* row_ptr, const uint32_t* col,
                          const uint32_t* o2n, const uint32_t* n2o, uint64_t* out_row_ptr,
                          uint32_t* out_col) {
    for (uint32_t v = 0; v < n; ++v)
        if (o2n[v] >= n || n2o[o2n[v]] != v)
            return fail(1, "apply_mapping: mapping is not a permutation");
    out_row_ptr[0] = 0;
    for (uint32_t v = 0; v < n; ++v) {
        uint32_t ov = n2o[v];
        uint64_t base = out_row_ptr[v], len = row_ptr[ov + 1] - row_ptr[ov];
        for (uint64_t k = 0; k < len; ++k) out_col[base + k] = o2n[col[row_ptr[ov] + k]];
        qsort(out_col + base, len, sizeof(uint32_t), cmp_u32);
        out_row_ptr[v + 1] = base + len;
    }
    return 0;
}

/* renumber.cpp:187-196 apply_mapping (EdgeList) */
int orc_apply_mapping_edges(uint32_t n, const uint32_t* edges, uint64_t e,
                            const uint32_t* o2n, const uint32_t* n2o, uint32_t* out) {
    (void)n;
    (void)n2o;
    for (uint64_t i = 0; i < 2 * e; ++i) out[i] = o2n[edges[i]];
    return 0;
}
