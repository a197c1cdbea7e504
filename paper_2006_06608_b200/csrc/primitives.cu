// Device-wide primitives used by preprocessing (scans, sorts, reductions).
// CUB from the CUDA toolkit; all calls are stream-ordered on the context
// stream with temporaries from the stream-ordered allocator.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include "gnna_common.cuh"

namespace {
__global__ void k_rebase_u64(uint64_t* v, uint64_t count, uint64_t base) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
        v[i] -= base;
}
}  // namespace

namespace gnna {

void rebase_u64(gnna_ctx* ctx, uint64_t* v, uint64_t count, uint64_t base) {
    if (!count) return;
    k_rebase_u64<<<grid_for(count, 256), 256, 0, ctx->stream>>>(v, count, base);
    launched(ctx, "k_rebase_u64");
}

uint64_t exclusive_scan_u64(gnna_ctx* ctx, const uint64_t* d_in, uint64_t* d_out, uint64_t count) {
    // d_out has count+1 entries; d_out[count] = total.
    if (count == 0) {
        GNNA_CUDA(cudaMemsetAsync(d_out, 0, sizeof(uint64_t), ctx->stream));
        return 0;
    }
    size_t bytes = 0;
    GNNA_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, d_in, d_out + 1, (int64_t)count, ctx->stream));
    DevBuf<uint8_t> tmp(bytes, ctx->stream);
    GNNA_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), bytes, d_in, d_out + 1, (int64_t)count, ctx->stream));
    GNNA_CUDA(cudaMemsetAsync(d_out, 0, sizeof(uint64_t), ctx->stream));
    uint64_t total = 0;
    to_host(ctx, &total, d_out + count, 1);
    return total;
}

uint64_t exclusive_scan_u32_to_u64(gnna_ctx* ctx, const uint32_t* d_in, uint64_t* d_out, uint64_t count) {
    if (count == 0) {
        GNNA_CUDA(cudaMemsetAsync(d_out, 0, sizeof(uint64_t), ctx->stream));
        return 0;
    }
    size_t bytes = 0;
    GNNA_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, d_in, d_out + 1, (int64_t)count, ctx->stream));
    DevBuf<uint8_t> tmp(bytes, ctx->stream);
    GNNA_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), bytes, d_in, d_out + 1, (int64_t)count, ctx->stream));
    GNNA_CUDA(cudaMemsetAsync(d_out, 0, sizeof(uint64_t), ctx->stream));
    uint64_t total = 0;
    to_host(ctx, &total, d_out + count, 1);
    return total;
}

uint64_t reduce_sum_u64(gnna_ctx* ctx, const uint64_t* d_in, uint64_t count) {
    if (count == 0) return 0;
    DevBuf<uint64_t> out(1, ctx->stream);
    size_t bytes = 0;
    GNNA_CUDA(cub::DeviceReduce::Sum(nullptr, bytes, d_in, out.get(), (int64_t)count, ctx->stream));
    DevBuf<uint8_t> tmp(bytes, ctx->stream);
    GNNA_CUDA(cub::DeviceReduce::Sum(tmp.get(), bytes, d_in, out.get(), (int64_t)count, ctx->stream));
    uint64_t total = 0;
    to_host(ctx, &total, out.get(), 1);
    return total;
}

void sort_pairs_u64_u32(gnna_ctx* ctx, uint64_t* keys, uint32_t* vals, uint64_t count, int end_bit) {
    if (count <= 1) return;
    DevBuf<uint64_t> k2(count, ctx->stream);
    DevBuf<uint32_t> v2(count, ctx->stream);
    cub::DoubleBuffer<uint64_t> kb(keys, k2.get());
    cub::DoubleBuffer<uint32_t> vb(vals, v2.get());
    size_t bytes = 0;
    GNNA_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kb, vb, (int64_t)count, 0, end_bit, ctx->stream));
    DevBuf<uint8_t> tmp(bytes, ctx->stream);
    GNNA_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, kb, vb, (int64_t)count, 0, end_bit, ctx->stream));
    if (kb.Current() != keys)
        GNNA_CUDA(cudaMemcpyAsync(keys, kb.Current(), count * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    if (vb.Current() != vals)
        GNNA_CUDA(cudaMemcpyAsync(vals, vb.Current(), count * 4, cudaMemcpyDeviceToDevice, ctx->stream));
}

void sort_keys_u64(gnna_ctx* ctx, uint64_t* keys, uint64_t count, int end_bit) {
    if (count <= 1) return;
    DevBuf<uint64_t> k2(count, ctx->stream);
    cub::DoubleBuffer<uint64_t> kb(keys, k2.get());
    size_t bytes = 0;
    GNNA_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, kb, (int64_t)count, 0, end_bit, ctx->stream));
    DevBuf<uint8_t> tmp(bytes, ctx->stream);
    GNNA_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(), bytes, kb, (int64_t)count, 0, end_bit, ctx->stream));
    if (kb.Current() != keys)
        GNNA_CUDA(cudaMemcpyAsync(keys, kb.Current(), count * 8, cudaMemcpyDeviceToDevice, ctx->stream));
}

}  // namespace gnna

namespace gnna {

__global__ void __launch_bounds__(1024) k_reduce_partials_narrow(const float* __restrict__ part, uint32_t chunks,
                                                                uint32_t total, float* __restrict__ out) {
    constexpr uint32_t OUTS = 8, SLICES = 128;
    __shared__ float red[SLICES][OUTS + 1];
    const uint32_t tx = threadIdx.x % OUTS, sl = threadIdx.x / OUTS;
    const uint32_t o = blockIdx.x * OUTS + tx;
    float s = 0.f;
    if (o < total) {
#pragma unroll 4
        for (uint32_t c = sl; c < chunks; c += SLICES) s += part[(size_t)c * total + o];
    }
    red[sl][tx] = s;
    __syncthreads();
    if (sl == 0 && o < total) {
        float t = 0.f;
        for (uint32_t i = 0; i < SLICES; ++i) t += red[i][tx];
        out[o] = t;
    }
}

void reduce_partials(gnna_ctx* ctx, const float* part, uint32_t chunks, uint32_t total, float* out) {
    static const int mode = [] {
        const char* e = std::getenv("GNNA_REDUCE_NARROW");  // A/B switch: 0 / 1 force either reducer
        return e && *e ? std::atoi(e) : -1;
    }();
    const bool narrow = mode >= 0 ? mode != 0 : ((total + 31) / 32 < (uint32_t)ctx->num_sms / 2 && chunks >= 256);
    if (narrow) {
        k_reduce_partials_narrow<<<(total + 7) / 8, 1024, 0, ctx->stream>>>(part, chunks, total, out);
        launched(ctx, "k_reduce_partials_narrow");
    } else {
        k_reduce_partials<<<(total + 31) / 32, 1024, 0, ctx->stream>>>(part, chunks, total, out);
        launched(ctx, "k_reduce_partials");
    }
}

}  // namespace gnna
