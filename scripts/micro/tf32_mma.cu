// Single-CTA check of tcgen05.mma kind::tf32 / kind::f16 with K-major and
// MN-major 128B-swizzled smem operands written by ordinary stores.
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include "../../paper_2109_10465_b200/csrc/tc_ptx.cuh"
using namespace moe::tc;
__device__ __forceinline__ uint32_t swz(int r, int c) { return r * 128 + ((c ^ (r & 7)) << 4); }

template <bool TF32, bool BMN>
__global__ void k(float* out, int variant) {
    __shared__ __align__(1024) uint8_t sm[32 * 1024];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x;
    // A: 128 rows x 128 B (K-major), value of A(m,k) = 1 + (m % 3) ; B: 64 x 128B value 1 (+k%2 for k-major)
    uint8_t* A = sm;
    uint8_t* B = sm + 16384;
    for (int q = tid; q < 128 * 8; q += blockDim.x) {
        int r = q / 8, c = q % 8;
        if (TF32) {
            float v = 1.f + (r % 3);
            *reinterpret_cast<float4*>(A + swz(r, c)) = make_float4(v, v, v, v);
        } else {
            __nv_bfloat16 v = __float2bfloat16(1.f + (r % 3));
            __nv_bfloat16 a[8] = {v, v, v, v, v, v, v, v};
            *reinterpret_cast<uint4*>(A + swz(r, c)) = *reinterpret_cast<uint4*>(a);
        }
    }
    for (int q = tid; q < 64 * 8; q += blockDim.x) {
        int r = q / 8, c = q % 8;
        if (TF32) *reinterpret_cast<float4*>(B + swz(r, c)) = make_float4(1.f, 1.f, 1.f, 1.f);
        else {
            __nv_bfloat16 v = __float2bfloat16(1.f);
            __nv_bfloat16 a[8] = {v, v, v, v, v, v, v, v};
            *reinterpret_cast<uint4*>(B + swz(r, c)) = *reinterpret_cast<uint4*>(a);
        }
    }
    if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (tid == 0) {
        uint32_t idesc;
        if (TF32) idesc = make_idesc_tf32(128, 64, 0, BMN ? 1 : 0);
        else idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((64 >> 3) << 17) | ((128 >> 4) << 24);
        if (variant == 1) idesc |= 0;  // placeholder
        const uint64_t ad = sdesc(smem_u32(A), 16, 1024);
        const uint64_t bd = BMN ? sdesc(smem_u32(B), 4096, 1024) : sdesc(smem_u32(B), 16, 1024);
        if (TF32) tc_mma_tf32(tmem, ad, bd, idesc, 0u);
        else tc_mma(tmem, ad, bd, idesc, 0u);
        tc_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    uint32_t v[32];
    tmem_ld32(tmem + ((uint32_t)((tid / 32) * 32) << 16), v);
    out[tid * 2] = __uint_as_float(v[0]);
    out[tid * 2 + 1] = __uint_as_float(v[5]);
    tc_fence_before();
    __syncthreads();
    if (tid < 32) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
    }
}
int main() {
    float* d; cudaMalloc(&d, 256 * 4);
    float h[256];
    auto run = [&](const char* nm, void (*kern)(float*, int)) {
        cudaMemset(d, 0xff, 256 * 4);
        kern<<<1, 128>>>(d, 0);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 256 * 4, cudaMemcpyDeviceToHost);
        printf("%-14s err=%d  row0 %g %g  row1 %g  row2 %g row100 %g\n", nm, (int)e, h[0], h[1], h[2], h[4], h[200]);
    };
    run("bf16 K/K", k<false, false>);
    run("tf32 K/K", k<true, false>);
    run("tf32 K/MN", k<true, true>);
    return 0;
}
