// Microbenchmark: cycles per 312-word block of the register warp twister,
// alone and with shared-memory publication.  nvcc -arch=sm_100a -O3.
#include <cstdio>
#include <cstdint>
constexpr uint64_t A = 0xB5026F5AA96619E9ULL, UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
__device__ __forceinline__ uint64_t mix(uint64_t lo_word, uint64_t hi_word) {
    const uint64_t y = (lo_word & UM) | (hi_word & LM);
    return (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
}
__device__ __forceinline__ void warp_twist(uint64_t (&Aw)[5], uint64_t (&Bw)[5], int lane) {
    const uint64_t a_next = __shfl_down_sync(0xffffffffu, Aw[0], 1);
    const uint64_t b_next = __shfl_down_sync(0xffffffffu, Bw[0], 1);
    const uint64_t o156 = __shfl_sync(0xffffffffu, Bw[0], 0);
    uint64_t nA[5];
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        uint64_t hi = r < 4 ? Aw[r + 1] : a_next;
        if (r == 0 && lane == 31) hi = o156;
        nA[r] = mix(Aw[r], hi) ^ Bw[r];
    }
    const uint64_t new0 = __shfl_sync(0xffffffffu, nA[0], 0);
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        uint64_t hi = r < 4 ? Bw[r + 1] : b_next;
        if (r == 0 && lane == 31) hi = new0;
        Bw[r] = mix(Bw[r], hi) ^ nA[r];
        Aw[r] = nA[r];
    }
}
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k_twist(int iters, int store, unsigned long long* out, uint64_t* sink) {
    __shared__ uint64_t ring[8 * 312];
    __shared__ uint64_t bar[2];
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[0])), "r"(store == 2 ? 32 : 1));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[1])), "r"(1));
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    if (threadIdx.x >= 32) return;
    uint64_t Aw[5], Bw[5];
    for (int r = 0; r < 5; ++r) { Aw[r] = lane * 77 + r; Bw[r] = lane * 13 + r * 5; }
    long long t0 = clock64();
    for (int b = 0; b < iters; ++b) {
        warp_twist(Aw, Bw, lane);
        if (store) {
            uint64_t* dst = ring + (b & 7) * 312 + lane * 5;
#pragma unroll
            for (int r = 0; r < 5; ++r)
                if (lane * 5 + r < 156) { dst[r] = Aw[r]; dst[r + 156] = Bw[r]; }
            __syncwarp();
            if (store == 2) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar[0])) : "memory");
            if (store == 3 && lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar[0])) : "memory");
            if (store == 4) {
                uint32_t ok;
                asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                             : "=r"(ok) : "r"(su32(&bar[1])), "r"(1u) : "memory");
                if (!ok) sink[0] = 1;
            }
        }
    }
    long long t1 = clock64();
    uint64_t x = 0;
    for (int r = 0; r < 5; ++r) x ^= Aw[r] ^ Bw[r];
    sink[threadIdx.x] = x ^ ring[lane];
    if (threadIdx.x == 0) out[0] = t1 - t0;
}
int main() {
    unsigned long long* d; uint64_t* s; cudaMalloc(&d, 8); cudaMalloc(&s, 8 * 1024);
    for (int store = 0; store < 5; ++store) {
        for (int threads : {32}) {
            k_twist<<<1, threads>>>(1000, store, d, s);
            k_twist<<<1, threads>>>(10000, store, d, s);
            unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("store=%d threads=%d: %.1f cycles/block\n", store, threads, h / 10000.0);
        }
    }
    return 0;
}
