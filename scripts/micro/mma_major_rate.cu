// tcgen05.mma kind::f16 issue rate with K-major vs MN-major smem operands:
// 148 CTAs, one thread issues NITER MMAs (M=128, N=256, K=16, bf16 -> fp32)
// into one TMEM accumulator from fixed 128B-swizzled tiles, then commits.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 mma_major_rate.cu -o mma_major_rate
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include "../../paper_2109_10465_b200/csrc/tc_ptx.cuh"
using namespace moe::tc;
constexpr int NITER = 4096;
__host__ __device__ constexpr uint32_t idesc_f16(uint32_t a_mn, uint32_t b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (a_mn << 15) | (b_mn << 16) | ((256 >> 3) << 17) | ((128 >> 4) << 24);
}
__global__ void __launch_bounds__(128) k(int a_mn, int b_mn, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x;
    for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (tid == 0) {
        const uint32_t sa = smem_u32(sm), sb = sa + 16384;
        const uint32_t idesc = idesc_f16(a_mn, b_mn);
        const long long c0 = clock64();
        for (int i = 0; i < NITER; ++i) {
            const int kk = i & 3;
            // A: 128 x 64 tile (K-major: 128 rows x 128 B; MN-major: 2 blocks of 64 M x 64 K rows)
            const uint64_t ad = a_mn ? sdesc(sa + kk * 2048, 8192, 1024) : sdesc(sa + kk * 32, 16, 1024);
            const uint64_t bd = b_mn ? sdesc(sb + kk * 2048, 8192, 1024) : sdesc(sb + kk * 32, 16, 1024);
            tc_mma(tmem, ad, bd, idesc, i ? 1u : 0u);
        }
        tc_commit(&bar);
        mbar_wait(&bar, 0);
        cyc[blockIdx.x] = clock64() - c0;
    }
    tc_fence_before();
    __syncthreads();
    if (tid < 32) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
    }
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 148 * 8);
    unsigned long long h[148];
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const char* nm[4] = {"A K / B K", "A K / B MN", "A MN / B K", "A MN / B MN"};
    for (int v = 0; v < 4; ++v) {
        const int a_mn = v >> 1, b_mn = v & 1;
        k<<<148, 128, 64 * 1024>>>(a_mn, b_mn, d);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<<<148, 128, 64 * 1024>>>(a_mn, b_mn, d);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i] / 148.0;
        const double flops = 2.0 * 128 * 256 * 16 * NITER * 148;
        printf("%-12s %.1f cycles/MMA, %.0f TFLOP/s (%s)\n", nm[v], avg / NITER, flops / (ms / 1e3) / 1e12,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
