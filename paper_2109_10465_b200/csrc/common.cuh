// common.cuh — shared device helpers for the B200 MoE layer kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

namespace moe {

constexpr int kNumSMs = 148;  // B200
constexpr int kRowAlign = 128; // expert segment rows are padded to the GEMM M tile

struct Status : std::runtime_error {
    int code;
    Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define MOE_CUDA_CHECK(expr)                                                                 \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess)                                                               \
            throw ::moe::Status(6, std::string(#expr) + ": " + cudaGetErrorString(_e));      \
    } while (0)

// Every kernel launch site calls MOE_LAUNCH_CHECK() right after the launch;
// it also counts launches (moe_kernel_launch_count, used by the bench).
uint64_t count_launch();
#define MOE_LAUNCH_CHECK()                        \
    do {                                          \
        MOE_CUDA_CHECK(cudaGetLastError());       \
        ::moe::count_launch();                    \
    } while (0)

// Programmatic dependent launch (PDL).  Kernels of the layer's main path are
// launched with programmatic stream serialisation, so a kernel's CTAs are
// scheduled (and run their independent prologue: barrier init, TMEM
// allocation, table loads) while the previous kernel drains.  Every kernel
// calls pdl_wait() before touching anything an earlier kernel wrote (it
// returns once the predecessor grid has completed and its writes are
// visible; a no-op for ordinary launches) and pdl_trigger() to let its own
// successor be scheduled.  MOE_B200_PDL=0 turns the attribute off.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_on();
template <class... P, class... A>
inline void launch_pdl(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_on() ? 1 : 0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MOE_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, static_cast<P>(args)...));
    ::moe::count_launch();
}

inline int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }
inline int64_t ceil_div(int64_t v, int64_t a) { return (v + a - 1) / a; }

// ---------------------------------------------------------------------------
// element IO: float or bf16 storage, fp32 math
// ---------------------------------------------------------------------------
__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
template <class T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) {
    return __float2bfloat16_rn(v);
}

// 16-byte vector of elements
template <class T> struct Vec16 {
    static constexpr int N = 16 / sizeof(T);
    union {
        uint4 u;
        T e[N];
    };
};

// V elements: a 16-byte vector when V * sizeof(T) == 16, else scalars.
template <class T, int V>
__device__ __forceinline__ void load_f(const T* __restrict__ p, float (&out)[V]) {
    if constexpr (V * sizeof(T) == 16) {
        Vec16<T> v;
        v.u = __ldg(reinterpret_cast<const uint4*>(p));
#pragma unroll
        for (int i = 0; i < V; ++i) out[i] = to_f(v.e[i]);
    } else {
#pragma unroll
        for (int i = 0; i < V; ++i) out[i] = to_f(p[i]);
    }
}

template <class T, int V>
__device__ __forceinline__ void store_f(T* __restrict__ p, const float (&in)[V]) {
    if constexpr (V * sizeof(T) == 16) {
        Vec16<T> v;
#pragma unroll
        for (int i = 0; i < V; ++i) v.e[i] = from_f<T>(in[i]);
        *reinterpret_cast<uint4*>(p) = v.u;
    } else {
#pragma unroll
        for (int i = 0; i < V; ++i) p[i] = from_f<T>(in[i]);
    }
}

template <class T, int V>
__device__ __forceinline__ void copy_vec(T* __restrict__ dst, const T* __restrict__ src) {
    if constexpr (V * sizeof(T) == 16) {
        *reinterpret_cast<uint4*>(dst) = __ldg(reinterpret_cast<const uint4*>(src));
    } else {
#pragma unroll
        for (int i = 0; i < V; ++i) dst[i] = src[i];
    }
}

template <class T, int V>
__device__ __forceinline__ void zero_vec(T* __restrict__ dst) {
    if constexpr (V * sizeof(T) == 16) {
        *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
    } else {
#pragma unroll
        for (int i = 0; i < V; ++i) dst[i] = from_f<T>(0.f);
    }
}

__host__ __device__ __forceinline__ int64_t round_up_dev(int64_t v, int64_t a) {
    return (v + a - 1) / a * a;
}

// Vector width usable for rows of length d of element type T.
template <class T> inline int vec_width(int64_t d) {
    constexpr int V = 16 / sizeof(T);
    return d % V == 0 ? V : 1;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ bool finite_f(float v) { return isfinite(v); }

// round-to-nearest (ties away) to tf32, as the tensor-core gate kernels read fp32 operands
__device__ __forceinline__ float tf32_rna_dev(float v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
}

}  // namespace moe
