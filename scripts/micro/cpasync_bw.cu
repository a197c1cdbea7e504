// Microbenchmark: streaming a row-major buffer through a shared-memory ring
// the way k6_dense_bwd does (4 CTAs x 256 threads per SM, S stages of R rows
// x 152 B = dy 88 B + z 64 B per row), with (a) per-thread 16-byte cp.async +
// wait_group + CTA barriers, or (b) one thread's cp.async.bulk per stage +
// mbarrier (TMA bulk path, no L1 miss tracking).  No compute: the bound of
// the copy machinery alone.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cpasync_bw cpasync_bw.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int R, int S>
__global__ void __launch_bounds__(256, 4) k_cpasync(const float* __restrict__ dy, const float* __restrict__ z,
                                                   uint32_t m, uint32_t rpc, float* sink) {
    extern __shared__ __align__(16) float sm[];
    float* sdy = sm;               // [S][R*22]
    float* sz = sm + S * R * 22;   // [S][R*16]
    const uint32_t t = threadIdx.x;
    const uint64_t r0c = (uint64_t)blockIdx.x * rpc;
    const uint64_t r1c = r0c + rpc < m ? r0c + rpc : m;
    const uint32_t nblk = r1c > r0c ? (uint32_t)((r1c - r0c + R - 1) / R) : 0;
    auto load = [&](uint32_t blk) {
        if (blk < nblk) {
            const uint32_t buf = blk % S;
            const uint64_t r0 = r0c + (uint64_t)blk * R;
            const uint32_t nr = (uint32_t)(r1c - r0 < R ? r1c - r0 : R);
            const float* s1 = dy + r0 * 22; float* d1 = sdy + buf * R * 22;
            for (uint32_t e = t; e < nr * 22 / 4; e += 256)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(d1 + 4 * e)), "l"(s1 + 4 * e) : "memory");
            const float* s2 = z + r0 * 16; float* d2 = sz + buf * R * 16;
            for (uint32_t e = t; e < nr * 16 / 4; e += 256)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(d2 + 4 * e)), "l"(s2 + 4 * e) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    float acc = 0.f;
    for (int s = 0; s < S - 1; ++s) load(s);
    for (uint32_t blk = 0; blk < nblk; ++blk) {
        load(blk + S - 1);
        asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
        __syncthreads();
        acc += sdy[(blk % S) * R * 22 + t % (R * 22)] + sz[(blk % S) * R * 16 + t % (R * 16)];
        __syncthreads();
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (acc == 12345.f) sink[0] = acc;
}

template <int R, int S>
__global__ void __launch_bounds__(256, 4) k_bulk(const float* __restrict__ dy, const float* __restrict__ z,
                                                uint32_t m, uint32_t rpc, float* sink) {
    extern __shared__ __align__(16) float sm[];
    __shared__ uint64_t full[S];
    float* sdy = sm;
    float* sz = sm + S * R * 22;
    const uint32_t t = threadIdx.x;
    const uint64_t r0c = (uint64_t)blockIdx.x * rpc;
    const uint64_t r1c = r0c + rpc < m ? r0c + rpc : m;
    const uint32_t nblk = r1c > r0c ? (uint32_t)((r1c - r0c + R - 1) / R) : 0;
    if (t == 0) {
        for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    auto load = [&](uint32_t blk) {  // thread 0
        if (blk >= nblk) return;
        const uint32_t buf = blk % S, bar = su32(&full[buf]);
        const uint64_t r0 = r0c + (uint64_t)blk * R;
        const uint32_t nr = (uint32_t)(r1c - r0 < R ? r1c - r0 : R);
        const uint32_t b1 = nr * 88 / 16 * 16, b2 = nr * 64;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(b1 + b2) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(sdy + buf * R * 22)), "l"(dy + r0 * 22), "r"(b1), "r"(bar) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(sz + buf * R * 16)), "l"(z + r0 * 16), "r"(b2), "r"(bar) : "memory");
    };
    float acc = 0.f;
    if (t == 0) for (int s = 0; s < S - 1; ++s) load(s);
    for (uint32_t blk = 0; blk < nblk; ++blk) {
        if (t == 0) load(blk + S - 1);
        const uint32_t bar = su32(&full[blk % S]), ph = (blk / S) & 1;
        const long long t0 = clock64();
        for (;;) {
            uint32_t done;
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(bar), "r"(ph) : "memory");
            if (done) break;
            if (clock64() - t0 > (1ll << 33)) __trap();  // never hang the device
        }
        acc += sdy[(blk % S) * R * 22 + t % (R * 22)] + sz[(blk % S) * R * 16 + t % (R * 16)];
        __syncthreads();
    }
    if (acc == 12345.f) sink[0] = acc;
}

template <class K>
void run(const char* name, K kern, int R, int S, const float* dy, const float* z, uint32_t m, int sms, float* sink) {
    const size_t smem = (size_t)S * R * 38 * 4;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const uint32_t ctas = 4 * sms;
    const uint32_t rpc = ((m + ctas - 1) / ctas + R - 1) / R * R;
    const uint32_t grid = (m + rpc - 1) / rpc;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(a);
        kern<<<grid, 256, smem>>>(dy, z, m, rpc, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep) best = ms < best ? ms : best;
    }
    const double bytes = (double)m * 152;
    printf("{\"kernel\": \"%s\", \"R\": %d, \"S\": %d, \"us\": %.2f, \"GBps\": %.0f, \"err\": \"%s\"}\n", name, R, S,
           best * 1e3, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint32_t m = 410236 * 8;  // 8x the C3 rows: 500 MB, beyond L2
    float *dy, *z, *sink;
    cudaMalloc(&dy, (size_t)m * 88); cudaMalloc(&z, (size_t)m * 64); cudaMalloc(&sink, 64);
    cudaMemset(dy, 0, (size_t)m * 88); cudaMemset(z, 0, (size_t)m * 64);
    run("cp.async", k_cpasync<64, 4>, 64, 4, dy, z, m, sms, sink);
    run("cp.async", k_cpasync<64, 6>, 64, 6, dy, z, m, sms, sink);
    run("bulk", k_bulk<64, 4>, 64, 4, dy, z, m, sms, sink);
    run("bulk", k_bulk<64, 6>, 64, 6, dy, z, m, sms, sink);
    run("bulk", k_bulk<128, 3>, 128, 3, dy, z, m, sms, sink);
    return 0;
}
