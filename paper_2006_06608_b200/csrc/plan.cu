// Preprocessing on the GPU: K1 (workload units, schedule.cpp:16-30) and K2
// (Algorithm 1, memplan.cpp:9-63), plus the run/carry layout the aggregation
// kernel consumes.  All integer outputs are bit-exact with the reference.
//
// Closed forms used (verified in the survey against the reference, and in
// tests/ against oracle/_ref):
//   units:  node v owns ceil(deg(v)/ngs) consecutive units starting at
//           ustart[v] = exclusive_scan(ceil(deg/ngs)); unit j of v covers
//           [row_ptr[v] + j*ngs, min(row_ptr[v] + (j+1)*ngs, row_ptr[v+1])).
//   leader: u % wpb == 0  or  target[u] != target[u-1]          (memplan.cpp:44-58)
//   slot:   (number of leaders in [floor(u/wpb)*wpb, u]) - 1     (memplan.cpp:44-60)
// One warp owns one schedule block (wpb <= 32): ballot + popc gives both.
#include "gnna_common.cuh"

namespace {

using gnna::DevBuf;

__global__ void k1_count(const uint64_t* __restrict__ row_ptr, uint32_t r0, uint32_t rows, uint32_t ngs,
                         uint64_t* __restrict__ cnt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t deg = row_ptr[r0 + i + 1] - row_ptr[r0 + i];
        cnt[i] = (deg + ngs - 1) / ngs;
    }
}

// One warp per node: lanes stride over the node's units.
__global__ void k1_write(const uint64_t* __restrict__ row_ptr, uint32_t r0, uint32_t rows, uint32_t ngs,
                         const uint64_t* __restrict__ ustart, uint64_t* __restrict__ part_ptr,
                         uint32_t* __restrict__ part2node) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t i = blockIdx.x * (uint64_t)(blockDim.x / 32) + threadIdx.x / 32; i < rows; i += warps) {
        const uint32_t v = r0 + (uint32_t)i;
        const uint64_t b = row_ptr[v];
        const uint64_t u0 = ustart[i], u1 = ustart[i + 1];
        for (uint64_t u = u0 + lane; u < u1; u += 32) {
            part_ptr[u] = b + (u - u0) * ngs;
            part2node[u] = v;
        }
    }
}

__global__ void k1_tail(const uint64_t* __restrict__ row_ptr, uint32_t r1, uint64_t G, uint64_t* part_ptr) {
    part_ptr[G] = row_ptr[r1];
}

// K2: one warp per schedule block of `wpb` units (wpb <= 32).
// Writes Algorithm-1 slot/leader (either may be null) and the kernel flags.
__global__ void k2_plan(const uint32_t* __restrict__ target, uint64_t G, uint32_t wpb,
                        uint8_t* __restrict__ slot, uint8_t* __restrict__ leader,
                        uint8_t* __restrict__ uflags, const uint64_t* __restrict__ ustart, uint32_t r0) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nblk = (G + wpb - 1) / wpb;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t sb = blockIdx.x * (uint64_t)(blockDim.x / 32) + threadIdx.x / 32; sb < nblk; sb += warps) {
        const uint64_t u = sb * wpb + lane;
        const bool in = lane < wpb && u < G;
        uint32_t t = 0, tprev = 0;
        if (in) {
            t = target[u];
            tprev = lane ? target[u - 1] : 0;
        }
        const bool start = in && (lane == 0 || t != tprev);
        const uint32_t starts = __ballot_sync(0xffffffffu, start);
        const uint32_t inmask = __ballot_sync(0xffffffffu, in);
        if (!in) continue;
        const uint32_t s = __popc(starts & ((2u << lane) - 1u)) - 1u;
        if (slot) slot[u] = (uint8_t)s;
        if (leader) leader[u] = start ? 1 : 0;
        if (uflags) {
            const bool last_in_block = lane == 31 || !((inmask >> (lane + 1)) & 1u);
            const bool run_end = last_in_block || ((starts >> (lane + 1)) & 1u);
            uint8_t f = (start ? UF_LEADER : 0) | (run_end ? UF_RUN_END : 0);
            const uint64_t a = ustart[t - r0], b = ustart[t - r0 + 1];
            if (a / wpb != (b - 1) / wpb) f |= UF_SPLIT;
            uflags[u] = f;
        }
    }
}

// Split-run carry slots: flag per unit = leader && split (scan -> cidx).
__global__ void k2_carry_flags(const uint8_t* __restrict__ uflags, uint64_t G, uint32_t* __restrict__ flag) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < G; u += (uint64_t)gridDim.x * blockDim.x)
        flag[u] = (uflags[u] & UF_LEADER) && (uflags[u] & UF_SPLIT) ? 1u : 0u;
}

__global__ void k2_u64_to_u32(const uint64_t* __restrict__ in, uint64_t n, uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = (uint32_t)in[i];
}

// Per row: packed (split << 32 | empty) indicator for the fix-up lists.
__global__ void k2_fix_flags(const uint64_t* __restrict__ ustart, uint32_t rows, uint32_t wpb,
                             uint64_t* __restrict__ packed) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a = ustart[i], b = ustart[i + 1];
        const uint64_t empty = (a == b) ? 1u : 0u;
        const uint64_t split = (a != b && a / wpb != (b - 1) / wpb) ? 1u : 0u;
        packed[i] = (split << 32) | empty;
    }
}

__global__ void k2_fix_lists(const uint64_t* __restrict__ ustart, uint32_t r0, uint32_t rows, uint32_t wpb,
                             const uint64_t* __restrict__ pos, uint64_t nsplit,
                             const uint32_t* __restrict__ cidx, uint32_t* __restrict__ nodes,
                             uint32_t* __restrict__ first, uint32_t* __restrict__ count) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a = ustart[i], b = ustart[i + 1];
        if (a == b) {
            nodes[nsplit + (pos[i] & 0xffffffffu)] = r0 + (uint32_t)i;
        } else if (a / wpb != (b - 1) / wpb) {
            const uint64_t k = pos[i] >> 32;
            nodes[k] = r0 + (uint32_t)i;
            first[k] = cidx[a];
            count[k] = (uint32_t)((b - 1) / wpb - a / wpb + 1);
        }
    }
}

// carry slot -> split-node index (the last-writer combine in K3 looks up
// its node's first slot and slot count through it).
__global__ void k2_carry_split(const uint32_t* __restrict__ first, const uint32_t* __restrict__ count, uint64_t nsplit,
                               uint32_t* __restrict__ carry_split) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nsplit; k += (uint64_t)gridDim.x * blockDim.x)
        for (uint32_t j = 0; j < count[k]; ++j) carry_split[first[k] + j] = (uint32_t)k;
}

// Consecutive-run validation for arbitrary targets (memplan.cpp:15-29):
// the first position whose target already had an earlier run.
__global__ void k2_first_run(const uint32_t* __restrict__ t, uint64_t G, unsigned long long* __restrict__ first) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < G; u += (uint64_t)gridDim.x * blockDim.x)
        if (u == 0 || t[u] != t[u - 1]) atomicMin(&first[t[u]], (unsigned long long)u);
}

__global__ void k2_violation(const uint32_t* __restrict__ t, uint64_t G, const unsigned long long* __restrict__ first,
                             unsigned long long* __restrict__ bad) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < G; u += (uint64_t)gridDim.x * blockDim.x)
        if ((u == 0 || t[u] != t[u - 1]) && first[t[u]] != u) atomicMin(bad, (unsigned long long)u);
}

__global__ void k_count_nonzero_u8(const uint8_t* __restrict__ f, uint64_t G, unsigned long long* __restrict__ out) {
    unsigned long long c = 0;
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < G; u += (uint64_t)gridDim.x * blockDim.x)
        c += f[u] != 0;
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, c);
}

__global__ void k_max_u32(const uint32_t* __restrict__ t, uint64_t G, unsigned* __restrict__ out) {
    unsigned m = 0;
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < G; u += (uint64_t)gridDim.x * blockDim.x)
        m = max(m, t[u]);
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

void validate(const gnna_params* p) {
    using gnna::raise;
    if (!p) raise(GNNA_ERR_DOMAIN, "null params");
    if (p->ngs < 1) raise(GNNA_ERR_DOMAIN, "params: ngs must be >= 1");
    if (p->tpw != 32) raise(GNNA_ERR_DOMAIN, "params: tpw is fixed at 32");
    if (p->dw < 1 || p->dw > p->tpw) raise(GNNA_ERR_DOMAIN, "params: dw must be in [1, tpw]");
    if (p->tpb == 0 || p->tpb % p->tpw != 0) raise(GNNA_ERR_DOMAIN, "params: tpb must be a positive multiple of tpw");
    if (p->tpb > 1024) raise(GNNA_ERR_DOMAIN, "params: tpb must be <= 1024");
    if (p->dim < 1) raise(GNNA_ERR_DOMAIN, "params: dim must be >= 1");
}

// Units per node and their exclusive scan (rows+1 entries). Returns G.
uint64_t unit_starts(gnna_ctx* ctx, const uint64_t* row_ptr, uint32_t r0, uint32_t rows, uint32_t ngs,
                     DevBuf<uint64_t>& ustart) {
    DevBuf<uint64_t> cnt(rows ? rows : 1, ctx->stream);
    ustart = DevBuf<uint64_t>((uint64_t)rows + 1, ctx->stream);
    if (rows) {
        k1_count<<<gnna::grid_for(rows, 256), 256, 0, ctx->stream>>>(row_ptr, r0, rows, ngs, cnt.get());
        gnna::launched(ctx, "k1_count");
    }
    return gnna::exclusive_scan_u64(ctx, cnt.get(), ustart.get(), rows);
}

}  // namespace

namespace gnna {
void validate_params(const gnna_params* p) { validate(p); }
}  // namespace gnna

extern "C" {

gnna_status gnna_validate_params(gnna_ctx* ctx, const gnna_params* p) {
    return gnna::guard(ctx, [&] { validate(p); });
}

gnna_status gnna_count_groups(gnna_ctx* ctx, const uint64_t* d_row_ptr, uint32_t n, uint32_t ngs,
                              uint64_t* num_groups) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (ngs < 1) gnna::raise(GNNA_ERR_DOMAIN, "partition_neighbors: ngs must be >= 1");
        DevBuf<uint64_t> us;
        *num_groups = unit_starts(ctx, d_row_ptr, 0, n, ngs, us);
    });
}

gnna_status gnna_partition_neighbors(gnna_ctx* ctx, const uint64_t* d_row_ptr, uint32_t n, uint32_t ngs,
                                     uint64_t* d_part_ptr, uint32_t* d_part2node) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (ngs < 1) gnna::raise(GNNA_ERR_DOMAIN, "partition_neighbors: ngs must be >= 1");
        DevBuf<uint64_t> us;
        const uint64_t G = unit_starts(ctx, d_row_ptr, 0, n, ngs, us);
        if (n) {
            k1_write<<<gnna::grid_for((uint64_t)n * 32, 256), 256, 0, ctx->stream>>>(d_row_ptr, 0, n, ngs, us.get(),
                                                                                      d_part_ptr, d_part2node);
            gnna::launched(ctx, "k1_write");
        }
        k1_tail<<<1, 1, 0, ctx->stream>>>(d_row_ptr, n, G, d_part_ptr);
        gnna::launched(ctx, "k1_tail");
    });
}

gnna_status gnna_build_mem_plan(gnna_ctx* ctx, const uint32_t* d_part2node, uint64_t G, const gnna_params* p,
                                uint8_t* d_slot, uint8_t* d_leader, uint64_t* shared_bytes) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        validate(p);
        const uint32_t wpb = p->tpb / p->tpw;
        if (G) {
            DevBuf<unsigned> mx(1, ctx->stream);
            GNNA_CUDA(cudaMemsetAsync(mx.get(), 0, 4, ctx->stream));
            k_max_u32<<<gnna::grid_for(G, 256, 4096), 256, 0, ctx->stream>>>(d_part2node, G, mx.get());
            gnna::launched(ctx, "k_max_u32");
            unsigned maxt = 0;
            gnna::to_host(ctx, &maxt, mx.get(), 1);
            DevBuf<unsigned long long> first((uint64_t)maxt + 1, ctx->stream);
            GNNA_CUDA(cudaMemsetAsync(first.get(), 0xff, ((uint64_t)maxt + 1) * 8, ctx->stream));
            DevBuf<unsigned long long> bad(1, ctx->stream);
            GNNA_CUDA(cudaMemsetAsync(bad.get(), 0xff, 8, ctx->stream));
            k2_first_run<<<gnna::grid_for(G, 256), 256, 0, ctx->stream>>>(d_part2node, G, first.get());
            gnna::launched(ctx, "k2_first_run");
            k2_violation<<<gnna::grid_for(G, 256), 256, 0, ctx->stream>>>(d_part2node, G, first.get(), bad.get());
            gnna::launched(ctx, "k2_violation");
            unsigned long long b = 0;
            gnna::to_host(ctx, &b, bad.get(), 1);
            if (b != ~0ull) {
                uint32_t node = 0;
                gnna::to_host(ctx, &node, d_part2node + b, 1);
                gnna::raise(GNNA_ERR_DOMAIN,
                            "build_mem_plan: warps of node " + std::to_string(node) + " are not consecutive");
            }
            const uint64_t blocks = (G + wpb - 1) / wpb;
            k2_plan<<<gnna::grid_for(blocks * 32, 256), 256, 0, ctx->stream>>>(d_part2node, G, wpb, d_slot, d_leader,
                                                                                nullptr, nullptr, 0);
            gnna::launched(ctx, "k2_plan");
        }
        if (shared_bytes) *shared_bytes = (uint64_t)wpb * p->dim * 4;
    });
}

gnna_status gnna_plan_create(gnna_ctx* ctx, const uint64_t* d_row_ptr, const uint32_t* d_col, uint32_t n,
                             uint32_t row_begin, uint32_t row_end, const gnna_params* p, int strategy,
                             gnna_plan** out) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        validate(p);
        if (row_begin > row_end || row_end > n) gnna::raise(GNNA_ERR_DOMAIN, "plan: bad row range");
        if (strategy < GNNA_NAIVE_ATOMIC || strategy > GNNA_WARP_SHARED)
            gnna::raise(GNNA_ERR_DOMAIN, "plan: unknown strategy");
        auto plan = new gnna_plan();
        try {
            cudaStream_t s = ctx->stream;
            plan->ctx = ctx;
            plan->params = *p;
            plan->strategy = strategy;
            plan->n = n;
            plan->row_begin = row_begin;
            plan->row_end = row_end;
            plan->row_ptr = d_row_ptr;
            plan->col = d_col;
            plan->wpb_params = p->tpb / p->tpw;
            // Naive/UnitSync flush every unit on its own: as values, a block of one unit.
            plan->wpb = strategy == GNNA_WARP_SHARED ? plan->wpb_params : 1;
            const uint32_t rows = row_end - row_begin;
            DevBuf<uint64_t> us;
            const uint64_t G = unit_starts(ctx, d_row_ptr, row_begin, rows, p->ngs, us);
            if (G >= (1ull << 32)) gnna::raise(GNNA_ERR_DOMAIN, "plan: more than 2^32 workload units");
            plan->G = G;
            plan->part_ptr = DevBuf<uint64_t>(G + 1, s);
            plan->part2node = DevBuf<uint32_t>(G ? G : 1, s);
            plan->slot = DevBuf<uint8_t>(G ? G : 1, s);
            plan->leader = DevBuf<uint8_t>(G ? G : 1, s);
            plan->uflags = DevBuf<uint8_t>(G ? G : 1, s);
            plan->cidx = DevBuf<uint32_t>(G ? G : 1, s);
            if (rows) {
                k1_write<<<gnna::grid_for((uint64_t)rows * 32, 256), 256, 0, s>>>(
                    d_row_ptr, row_begin, rows, p->ngs, us.get(), plan->part_ptr.get(), plan->part2node.get());
                gnna::launched(ctx, "k1_write");
            }
            k1_tail<<<1, 1, 0, s>>>(d_row_ptr, row_end, G, plan->part_ptr.get());
            gnna::launched(ctx, "k1_tail");
            {
                uint64_t ends[2] = {0, 0};
                GNNA_CUDA(cudaMemcpyAsync(&ends[0], d_row_ptr + row_begin, 8, cudaMemcpyDeviceToHost, s));
                GNNA_CUDA(cudaMemcpyAsync(&ends[1], d_row_ptr + row_end, 8, cudaMemcpyDeviceToHost, s));
                GNNA_CUDA(cudaStreamSynchronize(s));
                plan->nnz = ends[1] - ends[0];
            }
            if (G) {
                // Algorithm-1 arrays at the params' block width.
                const uint64_t b1 = (G + plan->wpb_params - 1) / plan->wpb_params;
                k2_plan<<<gnna::grid_for(b1 * 32, 256), 256, 0, s>>>(plan->part2node.get(), G, plan->wpb_params,
                                                                      plan->slot.get(), plan->leader.get(),
                                                                      plan->wpb == plan->wpb_params ? plan->uflags.get() : nullptr,
                                                                      us.get(), row_begin);
                gnna::launched(ctx, "k2_plan");
                if (plan->wpb != plan->wpb_params) {
                    const uint64_t b2 = (G + plan->wpb - 1) / plan->wpb;
                    k2_plan<<<gnna::grid_for(b2 * 32, 256), 256, 0, s>>>(plan->part2node.get(), G, plan->wpb, nullptr,
                                                                          nullptr, plan->uflags.get(), us.get(),
                                                                          row_begin);
                    gnna::launched(ctx, "k2_plan");
                }
                {  // Algorithm-1 runs = leaders at the params' block width
                    DevBuf<unsigned long long> cnt(1, s);
                    GNNA_CUDA(cudaMemsetAsync(cnt.get(), 0, 8, s));
                    k_count_nonzero_u8<<<gnna::grid_for(G, 256, 4096), 256, 0, s>>>(plan->leader.get(), G, cnt.get());
                    gnna::launched(ctx, "k_count_nonzero_u8");
                    unsigned long long r = 0;
                    gnna::to_host(ctx, &r, cnt.get(), 1);
                    plan->runs = r;
                }
                DevBuf<uint32_t> flag(G, s);
                k2_carry_flags<<<gnna::grid_for(G, 256), 256, 0, s>>>(plan->uflags.get(), G, flag.get());
                gnna::launched(ctx, "k2_carry_flags");
                DevBuf<uint64_t> pos(G + 1, s);
                plan->ncarry = gnna::exclusive_scan_u32_to_u64(ctx, flag.get(), pos.get(), G);
                k2_u64_to_u32<<<gnna::grid_for(G, 256), 256, 0, s>>>(pos.get(), G, plan->cidx.get());
                gnna::launched(ctx, "k2_u64_to_u32");
            }
            if (rows) {
                DevBuf<uint64_t> packed(rows, s), pos((uint64_t)rows + 1, s);
                k2_fix_flags<<<gnna::grid_for(rows, 256), 256, 0, s>>>(us.get(), rows, plan->wpb, packed.get());
                gnna::launched(ctx, "k2_fix_flags");
                const uint64_t tot = gnna::exclusive_scan_u64(ctx, packed.get(), pos.get(), rows);
                plan->nsplit = tot >> 32;
                plan->nempty = tot & 0xffffffffu;
                const uint64_t nfix = plan->nsplit + plan->nempty;
                plan->fix_nodes = DevBuf<uint32_t>(nfix ? nfix : 1, s);
                plan->fix_first = DevBuf<uint32_t>(plan->nsplit ? plan->nsplit : 1, s);
                plan->fix_count = DevBuf<uint32_t>(plan->nsplit ? plan->nsplit : 1, s);
                if (nfix) {
                    k2_fix_lists<<<gnna::grid_for(rows, 256), 256, 0, s>>>(us.get(), row_begin, rows, plan->wpb,
                                                                            pos.get(), plan->nsplit, plan->cidx.get(),
                                                                            plan->fix_nodes.get(), plan->fix_first.get(),
                                                                            plan->fix_count.get());
                    gnna::launched(ctx, "k2_fix_lists");
                }
            }
            if (plan->ncarry) plan->carry = DevBuf<uint8_t>(plan->ncarry * (uint64_t)p->dim * 8, s);
            plan->carry_split = DevBuf<uint32_t>(plan->ncarry ? plan->ncarry : 1, s);
            plan->split_cnt = DevBuf<uint32_t>(plan->nsplit ? plan->nsplit : 1, s);
            GNNA_CUDA(cudaMemsetAsync(plan->split_cnt.get(), 0, (plan->nsplit ? plan->nsplit : 1) * 4, s));
            if (plan->nsplit) {
                k2_carry_split<<<gnna::grid_for(plan->nsplit, 256), 256, 0, s>>>(
                    plan->fix_first.get(), plan->fix_count.get(), plan->nsplit, plan->carry_split.get());
                gnna::launched(ctx, "k2_carry_split");
            }
            GNNA_CUDA(cudaStreamSynchronize(s));
        } catch (...) {
            delete plan;
            throw;
        }
        *out = plan;
    });
}

void gnna_plan_destroy(gnna_plan* plan) { delete plan; }

gnna_status gnna_plan_info(const gnna_plan* plan, uint64_t* num_groups, uint64_t* num_runs,
                           uint64_t* num_split_nodes, uint64_t* num_carries) {
    return gnna::guard(nullptr, [&] {
        if (!plan) gnna::raise(GNNA_ERR_DOMAIN, "null plan");
        if (num_groups) *num_groups = plan->G;
        if (num_runs) *num_runs = plan->runs;
        if (num_split_nodes) *num_split_nodes = plan->nsplit;
        if (num_carries) *num_carries = plan->ncarry;
    });
}

gnna_status gnna_plan_arrays(const gnna_plan* plan, const uint64_t** d_part_ptr, const uint32_t** d_part2node,
                             const uint8_t** d_slot, const uint8_t** d_leader) {
    return gnna::guard(nullptr, [&] {
        if (!plan) gnna::raise(GNNA_ERR_DOMAIN, "null plan");
        if (d_part_ptr) *d_part_ptr = plan->part_ptr.get();
        if (d_part2node) *d_part2node = plan->part2node.get();
        if (d_slot) *d_slot = plan->slot.get();
        if (d_leader) *d_leader = plan->leader.get();
    });
}

}  // extern "C"
