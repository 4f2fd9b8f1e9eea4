// Microbenchmark: cycles per 312-word block of the register warp twister with
// shared-memory publication: conditional stores (as chunk_kernel) vs
// branch-free stores to a padded ring, vs inline-PTX shuffles.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 mt_micro2.cu
#include <cstdio>
#include <cstdint>
constexpr uint64_t A = 0xB5026F5AA96619E9ULL, UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
constexpr int N = 312, M = 156;
__device__ __forceinline__ uint64_t mix(uint64_t lo_word, uint64_t hi_word) {
    const uint64_t y = (lo_word & UM) | (hi_word & LM);
    return (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
}
__device__ __forceinline__ uint32_t shfl_idx(uint32_t v, int src) {
    uint32_t r;
    asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=r"(r) : "r"(v), "r"(src));
    return r;
}
__device__ __forceinline__ uint32_t shfl_down1(uint32_t v) {
    uint32_t r;
    asm volatile("shfl.sync.down.b32 %0, %1, 1, 0x1f, 0xffffffff;" : "=r"(r) : "r"(v));
    return r;
}
__device__ __forceinline__ uint64_t mk(uint32_t lo, uint32_t hi) { return ((uint64_t)hi << 32) | lo; }
template <int V>
__device__ __forceinline__ void warp_twist(uint64_t (&Aw)[5], uint64_t (&Bw)[5], int lane) {
    uint64_t a_next, b_next, o156, o0, o1;
    if (V < 2) {
        a_next = __shfl_down_sync(0xffffffffu, Aw[0], 1);
        b_next = __shfl_down_sync(0xffffffffu, Bw[0], 1);
        o156 = __shfl_sync(0xffffffffu, Bw[0], 0);
        o0 = __shfl_sync(0xffffffffu, Aw[0], 0);
        o1 = __shfl_sync(0xffffffffu, Aw[1], 0);
    } else {
        // only the bits mix() reads: hi word's low 63 bits, lo word's top bit
        a_next = mk(shfl_down1((uint32_t)Aw[0]), shfl_down1((uint32_t)(Aw[0] >> 32)));
        b_next = mk(shfl_down1((uint32_t)Bw[0]), shfl_down1((uint32_t)(Bw[0] >> 32)));
        o156 = mk(shfl_idx((uint32_t)Bw[0], 0), shfl_idx((uint32_t)(Bw[0] >> 32), 0));
        o0 = mk(0, shfl_idx((uint32_t)(Aw[0] >> 32), 0));
        o1 = mk(shfl_idx((uint32_t)Aw[1], 0), shfl_idx((uint32_t)(Aw[1] >> 32), 0));
    }
    uint64_t nA[5];
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        uint64_t hi = r < 4 ? Aw[r + 1] : a_next;
        if (r == 0 && lane == 31) hi = o156;
        nA[r] = mix(Aw[r], hi) ^ Bw[r];
    }
    const uint64_t new0 = mix(o0, o1) ^ o156;
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        uint64_t hi = r < 4 ? Bw[r + 1] : b_next;
        if (r == 0 && lane == 31) hi = new0;
        Bw[r] = mix(Bw[r], hi) ^ nA[r];
        Aw[r] = nA[r];
    }
}
template <int V, int G>
__global__ void k_twist(int iters, unsigned long long* out, uint64_t* sink) {
    __shared__ uint64_t ring[16 * N + 64];
    __shared__ uint64_t bars[32];
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 16) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[threadIdx.x])), "r"(32));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[16 + threadIdx.x])), "r"(1));
    }
    __syncthreads();
    if (G && (threadIdx.x >> 5) != 0) return;  // warp-uniform role split, as chunk_kernel
    uint64_t Aw[5], Bw[5];
    for (int r = 0; r < 5; ++r) { Aw[r] = lane * 77 + r; Bw[r] = lane * 13 + r * 5; }
    long long t0 = clock64();
    int slot = 0;
    for (int b = 0; b < iters; ++b) {
        warp_twist<V>(Aw, Bw, lane);
        if (V == 0) {
            uint64_t* dst = ring + slot * N + lane * 5;
#pragma unroll
            for (int r = 0; r < 5; ++r)
                if (lane * 5 + r < M) { dst[r] = Aw[r]; dst[r + M] = Bw[r]; }
        } else {
            // lane 31 words j = 156..159 land in the slot's tail / the next
            // slot's head (overwritten later) or the pad: no branch
            uint64_t* dst = ring + slot * N + lane * 5;
#pragma unroll
            for (int r = 0; r < 5; ++r) { dst[r] = Aw[r]; dst[r + M] = Bw[r]; }
        }
        if (V >= 3 && (V != 5 || (b & 1))) {
            const int fs = V == 5 ? slot >> 1 : slot;
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[fs])) : "memory");
        }
        if (V == 4) {
            uint32_t ok;
            asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(ok) : "r"((uint32_t)__cvta_generic_to_shared(&bars[16 + slot])), "r"(1u) : "memory");
            if (!ok) sink[0] = 1;
        }
        if (++slot == 16) slot = 0;
    }
    long long t1 = clock64();
    uint64_t x = 0;
    for (int r = 0; r < 5; ++r) x ^= Aw[r] ^ Bw[r];
    __syncwarp();
    sink[threadIdx.x & 31] = x ^ ring[lane * 7];
    if (threadIdx.x == 0) out[0] = t1 - t0;
}
template <int V, int G>
void run(unsigned long long* d, uint64_t* s) {
    k_twist<V, G><<<1, 64>>>(1000, d, s);
    k_twist<V, G><<<1, 64>>>(20000, d, s);
    unsigned long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("variant %d guard %d: %.1f cycles/block\n", V, G, h / 20000.0);
}
int main() {
    unsigned long long* d; uint64_t* s; cudaMalloc(&d, 8); cudaMalloc(&s, 8 * 1024);
    run<0, 0>(d, s); run<1, 0>(d, s); run<2, 0>(d, s); run<3, 0>(d, s); run<4, 0>(d, s); run<5, 0>(d, s);
    return 0;
}
