// DRAM read rate of the gate kernels' access pattern: 256 CTAs x 256
// threads, each CTA owning 128 rows x (d/4) columns of a [T][d] fp32 matrix
// and reading one 128-row x 32-column slab (128 B per row) per step, vs the
// same bytes read as contiguous 16 KB blocks (a tile-major layout).
#include <cstdio>
#include <cstdint>
__global__ void slab(const float4* __restrict__ a, int d, int ksplit, float* out) {
    const int tile = blockIdx.x / 4, split = blockIdx.x % 4;
    const int ac = threadIdx.x & 7, ar = threadIdx.x >> 3;
    float acc = 0.f;
    const int kper = d / ksplit;
    for (int k0 = split * kper; k0 < (split + 1) * kper; k0 += 32) {
        float4 v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = __ldg(a + ((int64_t)(tile * 128 + ar + 32 * i) * d + k0 + 4 * ac) / 4);
#pragma unroll
        for (int i = 0; i < 4; ++i) acc += v[i].x + v[i].y + v[i].z + v[i].w;
    }
    if (acc == 12345.f) out[0] = acc;
}
__global__ void blocks(const float4* __restrict__ a, int nblk_per_cta, float* out) {
    float acc = 0.f;
    for (int b = 0; b < nblk_per_cta; ++b) {
        const float4* p = a + ((int64_t)blockIdx.x * nblk_per_cta + b) * 1024;  // 16 KB blocks
        float4 v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = __ldg(p + threadIdx.x + 256 * i);
#pragma unroll
        for (int i = 0; i < 4; ++i) acc += v[i].x + v[i].y + v[i].z + v[i].w;
    }
    if (acc == 12345.f) out[0] = acc;
}
int main() {
    const int T = 8192, d = 2048, Q = 6;  // Q quarters of 67 MB > L2, read in rotation
    float* a0; float* o;
    cudaMalloc(&a0, (size_t)Q * T * d * 4); cudaMalloc(&o, 4);
    cudaMemset(a0, 0, (size_t)Q * T * d * 4);
    auto A = [&](int i) { return (const float4*)(a0 + (size_t)(i % Q) * T * d); };
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    slab<<<256, 256>>>(A(0), d, 4, o);
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) slab<<<256, 256>>>(A(i + 1), d, 4, o);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("slab pattern : %.1f us, %.0f GB/s\n", ms * 100, (double)T * d * 4 * 10 / (ms / 1e3) / 1e9);
    blocks<<<256, 256>>>(A(0), T * d / 4096 / 256, o);
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) blocks<<<256, 256>>>(A(i + 1), T * d / 4096 / 256, o);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("16KB blocks  : %.1f us, %.0f GB/s\n", ms * 100, (double)T * d * 4 * 10 / (ms / 1e3) / 1e9);
    return 0;
}
