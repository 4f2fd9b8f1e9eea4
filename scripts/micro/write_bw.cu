// HBM write-bandwidth ceilings on one GPU: vector stores (grid-stride, various
// grids) and TMA-style bulk stores (cp.async.bulk.global.shared::cta) from a
// shared-memory tile, to bound the write-dominated weight-gradient GEMMs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 write_bw.cu -o write_bw
#include <cstdio>
#include <cstdint>
__global__ void st_v4(uint4* p, size_t n16) {
    uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void st_bulk(uint8_t* p, size_t nbytes, int chunk) {
    extern __shared__ __align__(128) uint8_t sm[];
    for (int i = threadIdx.x; i < chunk / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
        for (size_t off = (size_t)blockIdx.x * chunk; off < nbytes; off += (size_t)gridDim.x * chunk) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + off), "r"(s), "r"(chunk) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}
int main() {
    size_t n = (size_t)4 << 30;
    uint8_t* p; cudaMalloc(&p, n);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int grid : {148, 296, 592, 1184, 4736}) for (int thr : {256, 1024}) {
        st_v4<<<grid, thr>>>((uint4*)p, n / 16);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) st_v4<<<grid, thr>>>((uint4*)p, n / 16);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("st.v4 grid %5d x %4d: %.0f GB/s\n", grid, thr, 5.0 * n / (ms / 1e3) / 1e9);
    }
    for (int chunk : {16384, 65536}) for (int grid : {148, 296}) {
        cudaFuncSetAttribute(st_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, chunk);
        st_bulk<<<grid, 128, chunk>>>(p, n, chunk);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) st_bulk<<<grid, 128, chunk>>>(p, n, chunk);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("bulk chunk %6d grid %4d: %.0f GB/s  (%s)\n", chunk, grid, 5.0 * n / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
