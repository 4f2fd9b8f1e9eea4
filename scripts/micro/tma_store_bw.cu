// Write ceiling of the weight-gradient GEMM's store pattern: 148 persistent
// CTAs, 4 warps each storing 32-row x 64-col bf16 boxes (128B-swizzled smem)
// with TMA tensor stores into a [rows x cols] bf16 matrix, tiles 128 x 256
// walked (m-tile, n-tile) with n fastest like grouped_gemm_kernel<WGRAD>.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tma_store_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__global__ void __launch_bounds__(128) store_tiles(const __grid_constant__ CUtensorMap tm, int MT, int NT, int bufs) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 4 * 4 * 4096 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    int cb = 0;
    for (int t = blockIdx.x; t < MT * NT; t += gridDim.x) {
        const int mt = t / NT, nt = t % NT;
        for (int c = 0; c < 256; c += 64) {
            uint8_t* sbuf = sm + (warp * 4 + (cb % bufs)) * 4096;
            if (lane == 0) {
                if (bufs == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                else asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                                 reinterpret_cast<uint64_t>(&tm)), "r"((uint32_t)__cvta_generic_to_shared(sbuf)),
                             "r"(nt * 256 + c), "r"(mt * 128 + warp * 32) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            __syncwarp();
            ++cb;
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
int main() {
    for (int shape = 0; shape < 2; ++shape) {
        const int64_t rows = shape == 0 ? 64LL * 8192 : 64LL * 2048, cols = shape == 0 ? 2048 : 8192;  // dW2, dW1
        void* p; cudaMalloc(&p, rows * cols * 2);
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
        cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
        cuuint32_t box[2] = {64, 32}, es[2] = {1, 1};
        CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, strides, box, es,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
        const int MT = rows / 128, NT = cols / 256;
        for (int grid : {148, 140, 136, 132, 128, 120, 112, 96, 64})
        for (int bufs : {2}) {
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaFuncSetAttribute(store_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
            store_tiles<<<grid, 128, 65536>>>(tm, MT, NT, bufs);
            cudaEventRecord(a);
            for (int k = 0; k < 5; ++k) store_tiles<<<grid, 128, 65536>>>(tm, MT, NT, bufs);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("%s grid %d bufs %d: %.3f ms per pass, %.0f GB/s (%s)\n", shape == 0 ? "dW2 [524288 x 2048]" : "dW1 [131072 x 8192]",
                   grid, bufs, ms / 5, 5.0 * rows * cols * 2 / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
        cudaFree(p);
    }
    return 0;
}
