// tcgen05.mma issue rate for the fused gate's shapes: kind::tf32 M=128 K=8 with
// N = 64 / 128 / 256, A from shared memory (SS) or from TMEM (TS), and
// kind::f16 M=128 N=64 K=16 for comparison.  148 CTAs, one thread issues NITER
// MMAs into one accumulator, then commits.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tf32_rate.cu -o tf32_rate
#include <cstdio>
#include <cstdint>
#include "../../paper_2109_10465_b200/csrc/tc_ptx.cuh"
using namespace moe::tc;
constexpr int NITER = 4096;
#ifndef STORE_SLEEP
#define STORE_SLEEP 0
#endif
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc, bool f16) {
    if (f16)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
    else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__host__ __device__ constexpr uint32_t idesc_f16(int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((128 >> 4) << 24);
}
template <bool F16, bool TS, int N, int UNR>
__global__ void __launch_bounds__(128) k(unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x;
    for (int i = tid; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (tid == 0) {
        const uint32_t sa = smem_u32(sm), sb = sa + 16384;
        constexpr uint32_t idesc = F16 ? idesc_f16(N) : make_idesc_tf32(128, N, 0, 0);
        const long long c0 = clock64();
        for (int i = 0; i < NITER; i += UNR) {
#pragma unroll
            for (int kk = 0; kk < UNR; ++kk) {
                const uint64_t bd = sdesc(sb + (kk & 3) * 32, 16, 1024);
                if (TS) {
                    mma_ts(tmem, tmem + 256 + (kk & 3) * 8, bd, idesc, (i | kk) ? 1u : 0u, F16);
                } else {
                    const uint64_t ad = sdesc(sa + (kk & 3) * 32, 16, 1024);
                    if (F16) tc_mma(tmem, ad, bd, idesc, (i | kk) ? 1u : 0u);
                    else tc_mma_tf32(tmem, ad, bd, idesc, (i | kk) ? 1u : 0u);
                }
            }
        }
        tc_commit(&bar);
        mbar_wait(&bar, 0);
        cyc[blockIdx.x] = clock64() - c0;
    }
    tc_fence_before();
    __syncthreads();
    if (tid < 32) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}
template <bool F16, bool TS, int N, int UNR>
void run(unsigned long long* d) {
    unsigned long long h[148];
    auto kf = k<F16, TS, N, UNR>;
    cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    kf<<<148, 128, 96 * 1024>>>(d);
    cudaDeviceSynchronize();
    kf<<<148, 128, 96 * 1024>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i] / 148.0;
    const int K = F16 ? 16 : 8;
    printf("%s %s N=%3d unroll %2d: %.1f cycles/MMA, %.0f MAC/clk (%s)\n", F16 ? "f16 " : "tf32", TS ? "TS" : "SS", N, UNR,
           avg / NITER, 128.0 * N * K / (avg / NITER), cudaGetErrorString(e));
}
// The fused gate's pattern: per K step of 8, three MMAs (hi.hi, hi.lo, lo.hi)
// into accumulator kk % 4 (N=64 columns each), A from TMEM at 256 + 64 * (step % 4);
// optionally warps 4..11 tcgen05.st 16 columns per lane in a loop meanwhile.
template <bool STORE>
__global__ void __launch_bounds__(384) kg(unsigned long long* cyc, int* stop) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    __shared__ volatile int done;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    if (tid == 0) { done = 0; mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    constexpr uint32_t idesc = make_idesc_tf32(128, 64, 0, 0);
    if (tid == 0) {
        const uint32_t sb = smem_u32(sm) + 16384;
        const long long c0 = clock64();
        for (int s = 0; s < NITER / 12; ++s) {
            const uint32_t ta = tmem + 256 + (s & 3) * 64;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const uint64_t bh = sdesc(sb + kk * 32, 16, 1024);
                const uint64_t bl = sdesc(sb + 8192 + kk * 32, 16, 1024);
                const uint32_t acc = tmem + kk * 64;
                mma_ts(acc, ta + kk * 8, bh, idesc, s ? 1u : 0u, false);
                mma_ts(acc, ta + kk * 8, bl, idesc, 1u, false);
                mma_ts(acc, ta + 32 + kk * 8, bh, idesc, 1u, false);
            }
        }
        tc_commit(&bar);
        mbar_wait(&bar, 0);
        cyc[blockIdx.x] = clock64() - c0;
        done = 1;
    } else if (STORE && warp >= 4) {
        uint32_t v[16];
        for (int i = 0; i < 16; ++i) v[i] = tid * 16 + i;
        const uint32_t ta = tmem + ((static_cast<uint32_t>(warp & 3) * 32) << 16) + 256 + 16 * ((warp - 4) >> 2);
        while (!done) {
            for (int j = 0; j < 4; ++j) {
                asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                             ::"r"(ta + j * 64), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                             "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
                asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                             ::"r"(ta + j * 64 + 32), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                             "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            }
            __nanosleep(STORE_SLEEP);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (tid < 32) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}
template <bool STORE>
void rung(unsigned long long* d) {
    unsigned long long h[148];
    auto kf = kg<STORE>;
    cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    kf<<<148, 384, 96 * 1024>>>(d, nullptr);
    cudaDeviceSynchronize();
    kf<<<148, 384, 96 * 1024>>>(d, nullptr);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i] / 148.0;
    printf("gate pattern (3 MMAs per kk, 4 accumulators) %s: %.1f cycles/MMA (%s)\n", STORE ? "with tcgen05.st traffic" : "alone",
           avg / (NITER / 12 * 12), cudaGetErrorString(e));
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 148 * 8);
    run<false, false, 64, 4>(d); run<false, false, 64, 16>(d); run<false, false, 128, 16>(d); run<false, false, 256, 16>(d);
    run<false, true, 64, 4>(d); run<false, true, 64, 16>(d); run<false, true, 128, 16>(d); run<false, true, 256, 16>(d);
    run<true, false, 64, 16>(d); run<true, false, 128, 16>(d); run<true, false, 256, 16>(d);
    run<true, true, 64, 16>(d); run<true, true, 256, 16>(d);
    rung<false>(d); rung<true>(d);
    return 0;
}
