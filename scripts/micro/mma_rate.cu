// Microbenchmark: tcgen05.mma issue-to-completion cost per instruction on one
// SM (one CTA per SM, one issuing thread), for the shapes the dense kernels
// use: kind::tf32 M = 128, N = 16..256, K = 8 per instruction, operands K-major
// SW128 (SS), MN-major SW128_BASE32B (SS), or A from TMEM (TS); kind::f16
// (bf16, K = 16) for comparison.  Smem contents are garbage (timing only).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_k(uint32_t addr) {  // K-major SW128
    return (uint64_t)((addr >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint64_t desc_mn(uint32_t addr, uint32_t lbo) {  // MN-major SW128_BASE32B
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) | ((uint64_t)(512 >> 4) << 32) |
           (1ull << 46) | (1ull << 61);
}
template <int N, int AMN, int BMN, int KIND>  // KIND 0 tf32, 1 bf16
__device__ constexpr uint32_t idesc() {
    return (1u << 4) | ((KIND == 0 ? 2u : 1u) << 7) | ((KIND == 0 ? 2u : 1u) << 10) | ((uint32_t)AMN << 15) |
           ((uint32_t)BMN << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// MODE 0: SS K-major, 1: SS MN-major, 2: TS (A in TMEM, B K-major)
template <int N, int MODE, int KIND, int NACC, int CEV = 0>
__global__ void __launch_bounds__(128, 1) k(int iters, long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar, bar2;
    __shared__ uint32_t slot;
    const uint32_t base = (su32(sm) + 1023u) & ~1023u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(su32(&bar2)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        constexpr uint32_t ID = idesc<N, MODE == 1 ? 1 : 0, MODE == 1 ? 1 : 0, KIND>();
        const uint32_t a = base, b = base + 64 * 1024;
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k8 = 0; k8 < 8; ++k8) {
                const uint32_t d = tmem + (uint32_t)((k8 % NACC) * N);
                const uint64_t da = MODE == 1 ? desc_mn(a + k8 * 1024, 8192) : desc_k(a + k8 * 32);
                const uint64_t db = MODE == 1 ? desc_mn(b + k8 * 1024, 8192) : desc_k(b + k8 * 32);
                const uint32_t acc = (it | k8) ? 1u : 0u;
                if (MODE == 3 || MODE == 4) {  // SS MN-major then TS, same (3) or other (4) accumulator
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                                 ::"r"(d), "l"(desc_mn(a + k8 * 1024, 8192)), "l"(desc_mn(b + k8 * 1024, 8192)), "r"(idesc<N, 1, 1, 0>()), "r"(acc));
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
                                 ::"r"(MODE == 3 ? d : d + 128u), "r"(tmem + 256u), "l"(desc_mn(b + k8 * 1024, 8192)), "r"(idesc<N, 0, 1, 0>()), "r"(acc));
                } else if (MODE == 2) {
                    if (KIND == 0)
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
                                     ::"r"(d), "r"(tmem + 256u), "l"(db), "r"(ID), "r"(acc));
                    else
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n"
                                     ::"r"(d), "r"(tmem + 256u), "l"(db), "r"(ID), "r"(acc));
                } else {
                    if (KIND == 0)
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                                     ::"r"(d), "l"(da), "l"(db), "r"(ID), "r"(acc));
                    else
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
                                     ::"r"(d), "l"(da), "l"(db), "r"(ID), "r"(acc));
                }
            }
            if (CEV && (it + 1) % CEV == 0 && it + 1 < iters)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2)) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
        asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W; }" ::"r"(su32(&bar)) : "memory");
        const long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int N, int MODE, int KIND, int NACC = 1, int CEV = 0>
void run(long long* d_out) {
    const int iters = 200, smem = 160 * 1024;
    cudaFuncSetAttribute(k<N, MODE, KIND, NACC, CEV>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<N, MODE, KIND, NACC, CEV><<<148, 128, smem>>>(iters, d_out);
    k<N, MODE, KIND, NACC, CEV><<<148, 128, smem>>>(iters, d_out);
    long long cyc = 0;
    cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaDeviceSynchronize();
    const double per = (double)cyc / (iters * 8 * (MODE >= 3 ? 2 : 1));
    const double kk = KIND == 0 ? 8 : 16;
    printf("{\"kind\": \"%s\", \"mode\": \"%s\", \"M\": 128, \"N\": %d, \"nacc\": %d, \"commit_every_16xmma\": %d, \"cyc_per_mma\": %.1f, \"macs_per_cyc\": %.0f, \"err\": \"%s\"}\n",
           KIND == 0 ? "tf32" : "bf16", MODE == 0 ? "SS-K" : MODE == 1 ? "SS-MN" : MODE == 2 ? "TS" : MODE == 3 ? "SS+TS same acc" : "SS+TS two acc", N, NACC, CEV, per, 128.0 * N * kk / per,
           cudaGetErrorString(e));
}

int main() {
    long long* d; cudaMalloc(&d, 64);
    run<32, 3, 0>(d); run<32, 3, 0, 1, 1>(d); run<32, 3, 0, 1, 2>(d); run<32, 3, 0, 1, 4>(d); run<32, 4, 0, 1, 1>(d);
    run<16, 0, 0>(d); run<32, 0, 0>(d); run<64, 0, 0>(d); run<128, 0, 0>(d); run<256, 0, 0>(d);
    run<32, 1, 0>(d); run<64, 1, 0>(d); run<128, 1, 0>(d); run<256, 1, 0>(d);
    run<16, 2, 0>(d); run<32, 2, 0>(d); run<64, 2, 0>(d); run<128, 2, 0>(d); run<256, 2, 0>(d);
    run<32, 0, 0, 4>(d); run<32, 1, 0, 4>(d);
    run<32, 0, 1>(d); run<128, 0, 1>(d); run<256, 0, 1>(d);
    return 0;
}
