// Pinned-host -> HBM copy rate alone and next to an HBM-saturating kernel:
// copy engine (cudaMemcpyAsync) vs an SM-driven zero-copy kernel on P CTAs
// (16-byte loads from mapped pinned memory, 8 in flight per thread).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 h2d_under_load.cu -o h2d_under_load
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void load_kernel(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n, int reps) {
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
            b[i] = a[i];
}
__global__ void __launch_bounds__(512) zc_copy(const uint4* __restrict__ h, uint4* __restrict__ d, size_t n) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n; i += 8 * stride) {
        uint4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = h[i + k * stride];
#pragma unroll
        for (int k = 0; k < 8; ++k) d[i + k * stride] = v[k];
    }
    for (; i < n; i += stride) d[i] = h[i];
}
int main() {
    const size_t bytes = 64ull << 20;  // 64 MB: one step's x + dy at config 3
    const size_t lbytes = 2ull << 30;
    void *hp, *dp, *la, *lb;
    CK(cudaHostAlloc(&hp, bytes, cudaHostAllocMapped));
    CK(cudaMalloc(&dp, bytes));
    CK(cudaMalloc(&la, lbytes));
    CK(cudaMalloc(&lb, lbytes));
    void* hdev;
    CK(cudaHostGetDevicePointer(&hdev, hp, 0));
    cudaStream_t s1, s2;
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int load = 0; load < 2; ++load) {
        for (int mode = 0; mode < 5; ++mode) {
            const int P = mode == 0 ? 0 : (mode == 1 ? 4 : mode == 2 ? 8 : mode == 3 ? 16 : 32);
            if (load) load_kernel<<<148 * 4, 512, 0, s2>>>((const uint4*)la, (uint4*)lb, lbytes / 32, 8);
            float best = 1e9;
            for (int it = 0; it < 5; ++it) {
                cudaEventRecord(e0, s1);
                if (P == 0) cudaMemcpyAsync(dp, hp, bytes, cudaMemcpyHostToDevice, s1);
                else zc_copy<<<P, 512, 0, s1>>>((const uint4*)hdev, (uint4*)dp, bytes / 16);
                cudaEventRecord(e1, s1);
                cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            CK(cudaDeviceSynchronize());
            printf("%s %s: %.1f GB/s\n", load ? "under HBM load" : "alone         ",
                   P == 0 ? "copy engine      " : (P == 4 ? "SM copy,  4 CTAs" : P == 8 ? "SM copy,  8 CTAs" : P == 16 ? "SM copy, 16 CTAs" : "SM copy, 32 CTAs"),
                   bytes / (best / 1e3) / 1e9);
        }
    }
    return 0;
}
