// optim.cu — the expert optimizer step on the device.
//
// AdamOptimizer::step (optim.cpp:21-57): optional global-norm clipping of all
// gradients, then per element
//   m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2;
//   theta -= lr * (m / bc1) / (sqrt(v / bc2) + eps),  bc_i = 1 - b_i^step.
// The reference keeps theta, m, v and the grads in f64.  Here theta (fp32
// master), m and v are fp32 in HBM and the update is evaluated in f64
// registers; bf16 weights for the next forward are written in the same pass.
// The kernel is HBM-bound: 4 B reads of theta/m/v, 2-4 B of grad, 4 B writes
// of theta/m/v and 2 B of the bf16 copy per parameter.
//
// The squared norm is a fixed-order two-level reduction in f64 (per-block
// partials over a fixed grid, then one block), accumulated tensor by tensor in
// stream order into a device double: deterministic.
#include <cmath>
#include <map>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace moe {
namespace opt {

constexpr int kNormBlocks = 4 * kNumSMs;
constexpr int kNormThreads = 256;

template <class T>
__device__ __forceinline__ double gval(const T* g, int64_t i) {
    return static_cast<double>(to_f(g[i]));
}

template <class T>
__global__ void __launch_bounds__(kNormThreads)
sqnorm_partials_kernel(const T* __restrict__ g, int64_t n, double* __restrict__ partials) {
    pdl_wait();
    pdl_trigger();
    __shared__ double s[kNormThreads];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kNormThreads + threadIdx.x; i < n;
         i += (int64_t)kNormBlocks * kNormThreads) {
        const double v = gval(g, i);
        acc += v * v;
    }
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int o = kNormThreads / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) partials[blockIdx.x] = s[0];
}

__global__ void __launch_bounds__(kNormThreads)
sqnorm_finalize_kernel(const double* __restrict__ partials, double* __restrict__ acc) {
    pdl_wait();
    pdl_trigger();
    __shared__ double s[kNormThreads];
    double a = 0.0;
    for (int i = threadIdx.x; i < kNormBlocks; i += kNormThreads) a += partials[i];
    s[threadIdx.x] = a;
    __syncthreads();
    for (int o = kNormThreads / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *acc += s[0];
}

__global__ void clip_scale_kernel(const double* __restrict__ sq, double clip, double* __restrict__ scale) {
    pdl_wait();
    pdl_trigger();
    // optim.cpp:26-37: scale = clip / ||g|| when clip > 0 and ||g|| > clip
    const double norm = sqrt(*sq);
    *scale = (clip > 0.0 && norm > clip) ? clip / norm : 1.0;
}

template <class G>
__global__ void __launch_bounds__(256)
adam_kernel(float* __restrict__ theta, float* __restrict__ m, float* __restrict__ v,
            const G* __restrict__ g, int64_t n, __nv_bfloat16* __restrict__ shadow,
            const double* __restrict__ scale_p, double lr, double b1, double b2, double eps,
            double bc1, double bc2) {
    pdl_wait();
    pdl_trigger();
    const double scale = scale_p ? *scale_p : 1.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double gi = gval(g, i) * scale;
        const double mi = b1 * static_cast<double>(m[i]) + (1.0 - b1) * gi;
        const double vi = b2 * static_cast<double>(v[i]) + (1.0 - b2) * gi * gi;
        const double th = static_cast<double>(theta[i]) - lr * (mi / bc1) / (sqrt(vi / bc2) + eps);
        m[i] = static_cast<float>(mi);
        v[i] = static_cast<float>(vi);
        theta[i] = static_cast<float>(th);
        if (shadow) shadow[i] = __float2bfloat16_rn(static_cast<float>(th));
    }
}

// Partial-sum scratch per (device, stream): concurrent norms on different
// streams (two optimizers, per-layer optimizers on side streams) never share
// a buffer; calls on one stream are ordered by the stream itself.
struct Scratch {
    std::map<std::pair<int, cudaStream_t>, double*> partials;
    std::mutex mu;
};
static Scratch& scratch() {
    static Scratch s;
    return s;
}
static double* partials_for(cudaStream_t st) {
    int dev = 0;
    MOE_CUDA_CHECK(cudaGetDevice(&dev));
    Scratch& s = scratch();
    std::lock_guard<std::mutex> lk(s.mu);
    double*& p = s.partials[{dev, st}];
    if (!p) MOE_CUDA_CHECK(cudaMalloc(&p, sizeof(double) * kNormBlocks));
    return p;
}

}  // namespace opt

void launch_grad_sqnorm(const void* g, int64_t n, bool bf16, double* acc, cudaStream_t st) {
    double* part = opt::partials_for(st);
    if (bf16)
        opt::sqnorm_partials_kernel<__nv_bfloat16><<<opt::kNormBlocks, opt::kNormThreads, 0, st>>>(
            static_cast<const __nv_bfloat16*>(g), n, part);
    else
        opt::sqnorm_partials_kernel<float><<<opt::kNormBlocks, opt::kNormThreads, 0, st>>>(
            static_cast<const float*>(g), n, part);
    MOE_LAUNCH_CHECK();
    opt::sqnorm_finalize_kernel<<<1, opt::kNormThreads, 0, st>>>(part, acc);
    MOE_LAUNCH_CHECK();
}

void launch_clip_scale(const double* sq, double clip, double* scale, cudaStream_t st) {
    opt::clip_scale_kernel<<<1, 1, 0, st>>>(sq, clip, scale);
    MOE_LAUNCH_CHECK();
}

void launch_adam(float* theta, float* m, float* v, const void* g, int64_t n, bool g_bf16,
                 __nv_bfloat16* shadow, const double* scale, double lr, double b1, double b2,
                 double eps, int64_t step, cudaStream_t st) {
    if (n <= 0) return;
    const double bc1 = 1.0 - std::pow(b1, static_cast<double>(step));
    const double bc2 = 1.0 - std::pow(b2, static_cast<double>(step));
    const int blocks = static_cast<int>(std::min<int64_t>(8 * kNumSMs, ceil_div(n, (int64_t)256)));
    if (g_bf16)
        opt::adam_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(
            theta, m, v, static_cast<const __nv_bfloat16*>(g), n, shadow, scale, lr, b1, b2, eps, bc1, bc2);
    else
        opt::adam_kernel<float><<<blocks, 256, 0, st>>>(theta, m, v, static_cast<const float*>(g), n, shadow,
                                                        scale, lr, b1, b2, eps, bc1, bc2);
    MOE_LAUNCH_CHECK();
}

}  // namespace moe
