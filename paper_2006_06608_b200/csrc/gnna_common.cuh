// Shared internals of libgnna (the CUDA side of include/gnna.h).  sm_100a only.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>

#include "gnna.h"

namespace gnna {
struct Staging;  // pinned bounce buffers + host copy threads for pageable transfers (capi.cu)
}

struct gnna_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    uint64_t launches = 0;
    int num_sms = 148;
    int l2_bytes = 0;
    int smem_optin = 0;
    gnna::Staging* staging = nullptr;  // created on the first large pageable copy
    ~gnna_ctx();
};

namespace gnna {

// Thrown inside entry points; converted to a status by `guard`.
struct Error {
    gnna_status code;
    std::string msg;
};

[[noreturn]] inline void raise(gnna_status code, std::string msg) { throw Error{code, std::move(msg)}; }

inline void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    if (e == cudaErrorMemoryAllocation) raise(GNNA_ERR_OOM, std::string(what) + ": out of device memory");
    raise(GNNA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define GNNA_CUDA(call) ::gnna::cuda_check((call), #call)

// Record + check a kernel launch on ctx.
inline void launched(gnna_ctx* ctx, const char* name) {
    ctx->launches++;
    cuda_check(cudaGetLastError(), name);
}

template <class F>
gnna_status guard(gnna_ctx* ctx, F&& f) {
    try {
        f();
        return GNNA_OK;
    } catch (const Error& e) {
        if (ctx) ctx->err = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        if (ctx) ctx->err = e.what();
        return GNNA_ERR_INTERNAL;
    }
}

inline void require_ctx(gnna_ctx* ctx) {
    if (!ctx) raise(GNNA_ERR_DOMAIN, "null gnna_ctx");
}

// Stream-ordered scratch buffer (cudaMallocAsync pool).
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(size_t count, cudaStream_t stream) : n(count), s(stream) {
        if (count) GNNA_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), stream));
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            reset();
            p = o.p; n = o.n; s = o.s;
            o.p = nullptr; o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { reset(); }
    // Frees on the allocation stream: that stream must outlive the buffer.
    void reset() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    // Frees ordered after the work queued so far on BOTH the allocation
    // stream and `cur` (the stream the buffer was last used on), so a buffer
    // that moved to another stream (gnna_set_stream) is not released under
    // work still queued there.  Not for use while `cur` is capturing.
    void release_on(cudaStream_t cur) {
        if (!p) return;
        if (cur != s) {
            cudaEvent_t e = nullptr;
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess) {
                cudaEventRecord(e, s);
                cudaStreamWaitEvent(cur, e, 0);
                cudaEventDestroy(e);
            }
            cudaFreeAsync(p, cur);
        } else {
            cudaFreeAsync(p, s);
        }
        p = nullptr;
        n = 0;
    }
    T* get() const { return p; }
};

inline unsigned grid_for(uint64_t work, unsigned block, uint64_t cap = 1u << 20) {
    uint64_t g = (work + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return static_cast<unsigned>(g);
}

template <class T>
inline void to_host(gnna_ctx* ctx, T* host, const T* dev, size_t count) {
    if (!count) return;
    GNNA_CUDA(cudaMemcpyAsync(host, dev, count * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
    GNNA_CUDA(cudaStreamSynchronize(ctx->stream));
}

// Exclusive scan (u64) over `count` values in place-compatible buffers; returns total.
uint64_t exclusive_scan_u64(gnna_ctx* ctx, const uint64_t* d_in, uint64_t* d_out, uint64_t count);
uint64_t exclusive_scan_u32_to_u64(gnna_ctx* ctx, const uint32_t* d_in, uint64_t* d_out, uint64_t count);
uint64_t reduce_sum_u64(gnna_ctx* ctx, const uint64_t* d_in, uint64_t count);
void sort_pairs_u64_u32(gnna_ctx* ctx, uint64_t* keys, uint32_t* vals, uint64_t count, int end_bit);
void sort_keys_u64(gnna_ctx* ctx, uint64_t* keys, uint64_t count, int end_bit);

// Deterministic sum of per-CTA partials part[chunks][total] -> out[total]
// (the split-row dW products).  A block covers 32 outputs x 32 chunk slices:
// loads are coalesced across outputs, each slice sums chunks s, s+32, ... in
// order, and slice 0 adds the 32 slice sums in slice order.  Fixed order for
// a given (chunks, total), with ~chunks/32 loads per thread in flight.
template <int SLICES = 32>
__global__ void __launch_bounds__(32 * SLICES) k_reduce_partials(const float* __restrict__ part, uint32_t chunks,
                                                                 uint32_t total, float* __restrict__ out) {
    __shared__ float red[SLICES][33];
    const uint32_t tx = threadIdx.x & 31, sl = threadIdx.x >> 5;
    const uint32_t o = blockIdx.x * 32 + tx;
    float s = 0.f;
    if (o < total) {
#pragma unroll 4
        for (uint32_t c = sl; c < chunks; c += SLICES) s += part[(size_t)c * total + o];
    }
    red[sl][tx] = s;
    __syncthreads();
    if (sl == 0 && o < total) {
        float t = 0.f;
#pragma unroll
        for (int i = 0; i < SLICES; ++i) t += red[i][tx];
        out[o] = t;
    }
}

// The same sum for few outputs over many chunks (the C3 dense backward:
// 352 outputs x ~600 CTA partials): 8 outputs x 128 chunk slices per block,
// so the grid has 4x the blocks and each slice's dependent chain is 4x
// shorter; slice 0 adds the 128 slice sums in slice order (fixed order).
__global__ void __launch_bounds__(1024) k_reduce_partials_narrow(const float* __restrict__ part, uint32_t chunks,
                                                                uint32_t total, float* __restrict__ out);

// Launches the better of the two reducers for (chunks, total).
void reduce_partials(gnna_ctx* ctx, const float* part, uint32_t chunks, uint32_t total, float* out);

}  // namespace gnna

// Internal plan (gnna_plan is opaque at the ABI).
struct gnna_plan {
    gnna_ctx* ctx = nullptr;
    gnna_params params{};
    int strategy = GNNA_WARP_SHARED;
    uint32_t n = 0, row_begin = 0, row_end = 0;
    uint32_t wpb = 1;            // Algorithm-1 block width (tpb/32; 1 for Naive/UnitSync flush)
    uint32_t wpb_params = 1;     // tpb/32 from params (counters use this)
    const uint64_t* row_ptr = nullptr;
    const uint32_t* col = nullptr;
    uint64_t G = 0;              // workload units
    uint64_t nnz = 0;            // CSR entries of the plan's rows
    uint64_t runs = 0;           // Algorithm-1 runs (= leaders)
    uint64_t nsplit = 0;         // nodes whose units span > 1 schedule block
    uint64_t ncarry = 0;         // carried run partials
    uint64_t nempty = 0;         // zero-degree rows in range
    gnna::DevBuf<uint64_t> part_ptr;   // G+1
    gnna::DevBuf<uint32_t> part2node;  // G
    gnna::DevBuf<uint8_t> slot;        // G, Algorithm-1 slot
    gnna::DevBuf<uint8_t> leader;      // G, Algorithm-1 leader flag
    gnna::DevBuf<uint8_t> uflags;      // G, kernel run flags (see plan.cu)
    gnna::DevBuf<uint32_t> cidx;       // G, carry index of a split run's leader
    gnna::DevBuf<uint32_t> fix_nodes;  // nsplit + nempty: split nodes then empty rows
    gnna::DevBuf<uint32_t> fix_first;  // nsplit: first carry index
    gnna::DevBuf<uint32_t> fix_count;  // nsplit: carries per split node
    mutable gnna::DevBuf<uint8_t> carry;  // ncarry * dim * 8 bytes (grown for wider dims)
    gnna::DevBuf<uint32_t> carry_split;   // ncarry: carry slot -> split-node index
    gnna::DevBuf<uint32_t> split_cnt;     // nsplit: K3 arrival counters (zero between launches)
};


// Unit flag bits (plan.cu builds them, aggregate.cu consumes them).
enum : uint8_t {
    UF_LEADER = 1,     // first unit of an Algorithm-1 run
    UF_RUN_END = 2,    // last unit of its run
    UF_SPLIT = 4,      // the unit's node spans more than one schedule block
};
