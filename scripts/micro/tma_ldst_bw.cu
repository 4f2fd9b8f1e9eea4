// The weight-gradient GEMM's memory traffic without the math: per 128x256
// output tile, a producer warp TMA-loads 2 x (16 KB A + 32 KB B) operand
// stages from an L2-resident buffer into a 3-stage ring while 4 warps TMA-store
// the 64 KB tile (32x64 boxes).  Compares stores alone vs stores + loads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tma_ldst_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void tma_ld(const CUtensorMap* m, uint64_t* bar, void* dst, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                 ::"r"(su(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(su(bar)), "r"(x), "r"(y) : "memory");
}
constexpr int kStages = 3, kStage = 49152;
__global__ void __launch_bounds__(160) k(const __grid_constant__ CUtensorMap tc, const __grid_constant__ CUtensorMap ta,
                                         int MT, int NT, int do_loads) {
    extern __shared__ __align__(1024) uint8_t smraw[];
    uint8_t* sm = smraw;
    uint8_t* stage = sm;                       // [3][48 KB]
    uint8_t* cst = sm + kStages * kStage;      // [4 warps][2][4 KB]
    __shared__ uint64_t full[kStages], empty[kStages];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) { for (int i = 0; i < kStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 4); } asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    for (int i = threadIdx.x; i < 8 * 4096 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(cst)[i] = i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (warp == 4) {  // producer
        if (lane == 0 && do_loads) {
            int s = 0; uint32_t ph = 0;
            for (int t = blockIdx.x; t < MT * NT; t += gridDim.x) {
                const int mt = t / NT, nt = t % NT;
                for (int kb = 0; kb < 2; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1);
                    expect_tx(&full[s], kStage);
                    for (int j = 0; j < 6; ++j)  // 2 x {64, 64} A boxes + 4 B boxes, 8 KB each
                        tma_ld(&ta, &full[s], stage + s * kStage + j * 8192, ((mt % 16) * 2 + (j < 2 ? j : 0)) * 64 % 2048, kb * 64 + (j >= 2 ? 128 : 0) + (nt % 4) * 256);
                    if (++s == kStages) { s = 0; ph ^= 1; }
                }
            }
        }
        return;
    }
    int s = 0; uint32_t ph = 0, cb = 0;
    for (int t = blockIdx.x; t < MT * NT; t += gridDim.x) {
        const int mt = t / NT, nt = t % NT;
        if (do_loads) for (int kb = 0; kb < 2; ++kb) {  // consume the operand stages
            mbar_wait(&full[s], ph);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == kStages) { s = 0; ph ^= 1; }
        }
        for (int c = 0; c < 256; c += 64) {
            uint8_t* sbuf = cst + (warp * 2 + (cb & 1)) * 4096;
            if (lane == 0) {
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                                 reinterpret_cast<uint64_t>(&tc)), "r"(su(sbuf)), "r"(nt * 256 + c), "r"(mt * 128 + warp * 32) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            __syncwarp();
            ++cb;
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
static CUtensorMap mk(void* p, int64_t rows, int64_t cols, int bc, int br) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br}, es[2] = {1, 1};
    if (cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        printf("encode failed\n");
    return tm;
}
int main() {
    const int64_t rows = 64LL * 8192, cols = 2048;  // dW2 shape
    void *c, *a;
    cudaMalloc(&c, rows * cols * 2);
    cudaMalloc(&a, 2048LL * 2048 * 2);  // 8 MB operand pool (L2 resident)
    CUtensorMap tc = mk(c, rows, cols, 64, 32), ta = mk(a, 2048, 2048, 64, 64);
    const int smem = kStages * kStage + 8 * 4096;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int loads = 0; loads < 2; ++loads) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        k<<<148, 160, smem>>>(tc, ta, rows / 128, cols / 256, loads);
        cudaEventRecord(e0);
        for (int i = 0; i < 5; ++i) k<<<148, 160, smem>>>(tc, ta, rows / 128, cols / 256, loads);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("loads %d: %.3f ms per pass, stores %.0f GB/s (%s)\n", loads, ms / 5, 5.0 * rows * cols * 2 / (ms / 1e3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
