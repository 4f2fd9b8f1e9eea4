// Cost of the weight-gradient epilogue's SM-side work on top of its TMA
// stores: 148 persistent CTAs x 4 warps write [rows x cols] bf16 in 128 x 256
// tiles (32 x 64 boxes, 128B swizzle) like grouped_gemm_kernel<WGRAD>.
//   mode 0  TMA stores of stale staging buffers (store ceiling)
//   mode 1  + per 64-column chunk: 32 cvt/pack, 8 STS.128, fence.proxy.async (current epilogue)
//   mode 2  + the same STS per chunk, one fence per tile (4 chunks, 8 staging buffers per warp)
//   mode 3  as 2 with 4 staging buffers per warp (one tile; wait for its reads before the next)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 epi_bw.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__global__ void __launch_bounds__(128) k(const __grid_constant__ CUtensorMap tm, int MT, int NT, int mode) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int cb = 0;
    float seed = lane * 0.001f + blockIdx.x;
    for (int t = blockIdx.x; t < MT * NT; t += gridDim.x) {
        const int mt = t / NT, nt = t % NT;
        for (int c = 0; c < 256; c += 64) {
            const int nb = mode == 2 ? 8 : mode == 3 ? 4 : 2;
            uint8_t* sbuf = sm + (warp * 8 + (cb % nb)) * 4096;
            if (mode >= 2 ? (c == 0) : true) {
                if (lane == 0) {
                    if (mode == 2) asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
                    else if (mode == 3) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                }
                __syncwarp();
            }
            if (mode >= 1) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    uint4 u;
                    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
                    for (int j = 0; j < 4; ++j) h2[j] = __floats2bfloat162_rn(seed + q * 8 + 2 * j, seed + c + j);
                    sts128(su(sbuf) + lane * 128 + ((q ^ (lane & 7)) << 4), u);
                }
                if (mode == 1 || c == 192) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                }
            }
            if (mode < 2 || c == 192) {
                const int n0 = mode >= 2 ? 0 : c, n1 = mode >= 2 ? 256 : c + 64;
                if (lane == 0) {
                    for (int cc = n0; cc < n1; cc += 64) {
                        uint8_t* b = mode >= 2 ? sm + (warp * 8 + ((cb - (c - cc) / 64) % nb)) * 4096 : sbuf;
                        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                                         reinterpret_cast<uint64_t>(&tm)), "r"(su(b)), "r"(nt * 256 + cc), "r"(mt * 128 + warp * 32)
                                     : "memory");
                    }
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
                __syncwarp();
            }
            ++cb;
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
int main() {
    const int64_t rows = 64LL * 8192, cols = 2048;
    void* p; cudaMalloc(&p, rows * cols * 2);
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, 32}, es[2] = {1, 1};
    cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = 4 * 8 * 4096;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int grid : {148, 128})
    for (int mode = 0; mode < 4; ++mode) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        k<<<grid, 128, smem>>>(tm, rows / 128, cols / 256, mode);
        cudaEventRecord(a);
        for (int i = 0; i < 5; ++i) k<<<grid, 128, smem>>>(tm, rows / 128, cols / 256, mode);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("grid %d mode %d: %.3f ms per pass, %.0f GB/s (%s)\n", grid, mode, ms / 5, 5.0 * rows * cols * 2 / (ms / 1e3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
