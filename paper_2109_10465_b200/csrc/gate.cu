// gate.cu — the gate's three GEMM-shaped steps, register-tiled fp32 FFMA.
//
//   logits = (x * noise) Wg                  routing.cpp:62-71 (mul + matmul)
//   dx     = (dL Wg^T) * noise               matmul bwd (ops.cpp:137-138) + mul bwd
//            + sum_k dX[row_k] (+ dy)        (ops.cpp:223-228), fused with the
//                                            dispatch bwd (routing.cpp:245-253) and
//                                            the combine residual bwd (routing.cpp:337-342)
//   dWg    = (x * noise)^T dL                matmul bwd (ops.cpp:140-143), split over
//                                            tokens, fixed-order reduction
//
// The gate has N = E <= 64 columns, far too narrow for a 128x256 tensor-core
// tile, and decision parity with the f64 oracle needs fp32-accurate logits
// (bf16/tf32 operands would flip near-ties), so these run on the FMA pipes
// with 64x64 (or 64x128) CTA tiles, 4x4 / 4x8 register micro-tiles and
// 16-byte vector loads.  The noise multiply happens while staging x.
#include "common.cuh"
#include "kernels.h"

namespace moe {

namespace gate {

constexpr int BT = 64, BE = 64, BK = 32, NT = 256;

template <class TX>
__device__ __forceinline__ void load8(const TX* p, float (&v)[8]) {
    if constexpr (sizeof(TX) == 2) {
        load_f<TX, 8>(p, v);
    } else {
        float a[4], b[4];
        load_f<TX, 4>(p, a);
        load_f<TX, 4>(p + 4, b);
#pragma unroll
        for (int i = 0; i < 4; ++i) { v[i] = a[i]; v[4 + i] = b[i]; }
    }
}

__device__ __forceinline__ void load8f(const float* p, float (&v)[8]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    const float4 b = __ldg(reinterpret_cast<const float4*>(p + 4));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// logits[T, E]: CTA = 64 tokens x 64 experts; thread = 4 tokens x 4 experts.
// Requires d % 32 == 0 and E % 4 == 0 (checked by the launcher).
template <class TX>
__global__ void __launch_bounds__(NT)
logits_kernel(const TX* __restrict__ x, const float* __restrict__ noise,
              const float* __restrict__ wg, float* __restrict__ logits, int64_t T, int d, int E,
              int k_per_split) {
    pdl_wait();
    pdl_trigger();
    __shared__ __align__(16) float Xs[BK][BT + 4];
    __shared__ __align__(16) float Ws[BK][BE + 4];
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    const int64_t t0 = (int64_t)blockIdx.x * BT;
    const int e0 = blockIdx.y * BE;
    const int kb = blockIdx.z * k_per_split, ke = min(d, kb + k_per_split);
    logits += (int64_t)blockIdx.z * T * E;  // split-K partials, summed in fixed order by softmax
    float acc[4][4] = {};
    // staging roles: x: 64 rows x 4 groups of 8 k; W: 32 rows x 16 float4
    const int xr = tid / 4, xq = tid % 4;
    for (int k0 = kb; k0 < ke; k0 += BK) {
        {
            float v[8];
            const int64_t t = t0 + xr;
            if (t < T) {
                load8<TX>(x + t * d + k0 + xq * 8, v);
                if (noise) {
                    float n[8];
                    load8f(noise + t * d + k0 + xq * 8, n);
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[i] *= n[i];
                }
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = 0.f;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) Xs[xq * 8 + i][xr] = v[i];
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int idx = tid + i * NT;  // 512 float4 = 32 x 16
            const int kr = idx / 16, c4 = idx % 16;
            const int e = e0 + c4 * 4;
            float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
            if (e < E) w = __ldg(reinterpret_cast<const float4*>(wg + (int64_t)(k0 + kr) * E + e));
            *reinterpret_cast<float4*>(&Ws[kr][c4 * 4]) = w;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            const float4 a = *reinterpret_cast<const float4*>(&Xs[k][ty * 4]);
            const float4 b = *reinterpret_cast<const float4*>(&Ws[k][tx * 4]);
            const float av[4] = {a.x, a.y, a.z, a.w};
            const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t t = t0 + ty * 4 + i;
        const int e = e0 + tx * 4;
        if (t < T && e < E)
            *reinterpret_cast<float4*>(logits + t * E + e) =
                make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    }
}

// dx tile: 64 tokens x 64 columns, K = E staged whole (E <= 64).
constexpr int DJ = 64, MAXE = 64;

template <class TIO>
__global__ void __launch_bounds__(NT)
dx_kernel(int64_t T, int d, int E, int K, int cap_pad, const float* __restrict__ dL,
          const float* __restrict__ wg, const float* __restrict__ noise, const TIO* __restrict__ dX,
          const int32_t* __restrict__ choice, const int32_t* __restrict__ pos,
          const TIO* __restrict__ dy, bool residual_is_x, TIO* __restrict__ dx,
          TIO* __restrict__ dres) {
    pdl_wait();
    pdl_trigger();
    __shared__ __align__(16) float Ls[MAXE][BT + 4];
    __shared__ __align__(16) float Wt[MAXE][DJ + 4];
    __shared__ int64_t rows[BT][2];
    __shared__ int anyk[BT];
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;  // 16 x 4 columns, 16 x 4 tokens
    const int64_t t0 = (int64_t)blockIdx.x * BT;
    const int j0 = blockIdx.y * DJ;
    for (int i = tid; i < BT * E; i += NT) {
        const int tt = i / E, e = i % E;
        const int64_t t = t0 + tt;
        Ls[e][tt] = t < T ? dL[t * E + e] : 0.f;
    }
    for (int i = tid; i < DJ * E; i += NT) {
        const int jj = i / E, e = i % E;
        Wt[e][jj] = wg[(int64_t)(j0 + jj) * E + e];
    }
    if (tid < BT) {
        const int64_t t = t0 + tid;
        int any = 0;
        for (int k = 0; k < 2; ++k) {
            int64_t r = -1;
            if (t < T && k < K) {
                const int32_t p = pos[t * K + k];
                if (p >= 0) {
                    r = (int64_t)choice[t * K + k] * cap_pad + p;
                    any = 1;
                }
            }
            rows[tid][k] = r;
        }
        anyk[tid] = any;
    }
    __syncthreads();
    float acc[4][4] = {};
    for (int e = 0; e < E; ++e) {
        const float4 a = *reinterpret_cast<const float4*>(&Ls[e][ty * 4]);
        const float4 b = *reinterpret_cast<const float4*>(&Wt[e][tx * 4]);
        const float av[4] = {a.x, a.y, a.z, a.w};
        const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[i][q] = fmaf(av[i], bv[q], acc[i][q]);
    }
    const int j = j0 + tx * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int tt = ty * 4 + i;
        const int64_t t = t0 + tt;
        if (t >= T) continue;
        float v[4];
        if (noise) {
            const float4 n = __ldg(reinterpret_cast<const float4*>(noise + t * d + j));
            v[0] = acc[i][0] * n.x; v[1] = acc[i][1] * n.y; v[2] = acc[i][2] * n.z; v[3] = acc[i][3] * n.w;
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = acc[i][q];
        }
        for (int k = 0; k < K; ++k) {
            const int64_t r = rows[tt][k];
            if (r < 0) continue;
            float g[4];
            load_f<TIO, 4>(dX + r * d + j, g);
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] += g[q];
        }
        if (!anyk[tt]) {
            float g[4];
            load_f<TIO, 4>(dy + t * d + j, g);
            if (residual_is_x) {
#pragma unroll
                for (int q = 0; q < 4; ++q) v[q] += g[q];
            } else if (dres) {
                store_f<TIO, 4>(dres + t * d + j, g);
            }
        } else if (!residual_is_x && dres) {
            float z[4] = {0.f, 0.f, 0.f, 0.f};
            store_f<TIO, 4>(dres + t * d + j, z);
        }
        store_f<TIO, 4>(dx + t * d + j, v);
    }
}

// dWg partials: part[s][j][e] = sum_{t in split s} x[t,j] noise[t,j] dL[t,e].
// CTA = 64 j x 64 e; K = tokens, 32 at a time (rows of x and dL are contiguous
// in j and e, so both tiles stage without transposes).
template <class TX>
__global__ void __launch_bounds__(NT)
dw_kernel(const TX* __restrict__ x, const float* __restrict__ noise,
          const float* __restrict__ dL, float* __restrict__ part, int64_t T, int d, int E,
          int64_t t_per_split) {
    pdl_wait();
    pdl_trigger();
    __shared__ __align__(16) float As[BK][BT + 4];  // [token][j]
    __shared__ __align__(16) float Bs[BK][BE + 4];  // [token][e]
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    const int j0 = blockIdx.x * BT, e0 = blockIdx.y * BE;
    const int64_t tb = (int64_t)blockIdx.z * t_per_split;
    const int64_t te = min(T, tb + t_per_split);
    float acc[4][4] = {};
    const int ar = tid / 8, aq = tid % 8;  // 32 tokens x 8 groups of 8 j
    for (int64_t k0 = tb; k0 < te; k0 += BK) {
        {
            float v[8];
            const int64_t t = k0 + ar;
            if (t < te) {
                load8<TX>(x + t * d + j0 + aq * 8, v);
                if (noise) {
                    float n[8];
                    load8f(noise + t * d + j0 + aq * 8, n);
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[i] *= n[i];
                }
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = 0.f;
            }
            *reinterpret_cast<float4*>(&As[ar][aq * 8]) = make_float4(v[0], v[1], v[2], v[3]);
            *reinterpret_cast<float4*>(&As[ar][aq * 8 + 4]) = make_float4(v[4], v[5], v[6], v[7]);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int idx = tid + i * NT;
            const int kr = idx / 16, c4 = idx % 16;
            const int64_t t = k0 + kr;
            const int e = e0 + c4 * 4;
            float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
            if (t < te && e < E) w = __ldg(reinterpret_cast<const float4*>(dL + t * E + e));
            *reinterpret_cast<float4*>(&Bs[kr][c4 * 4]) = w;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            const float4 a = *reinterpret_cast<const float4*>(&As[k][ty * 4]);
            const float4 b = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
            const float av[4] = {a.x, a.y, a.z, a.w};
            const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[i][q] = fmaf(av[i], bv[q], acc[i][q]);
        }
        __syncthreads();
    }
    float* P = part + (int64_t)blockIdx.z * d * E;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int jj = j0 + ty * 4 + i;
        const int e = e0 + tx * 4;
        if (e < E)
            *reinterpret_cast<float4*>(P + (int64_t)jj * E + e) =
                make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    }
}

}  // namespace gate

bool gate_fast_ok(int d, int E) { return d % 64 == 0 && E % 4 == 0 && E <= gate::MAXE; }

int gate_logit_splits(int64_t T, int d, int E) {
    const int64_t ctas = ceil_div(T, gate::BT) * ceil_div(E, gate::BE);
    int s = 1;
    while (s < kMaxGateSplits && ctas * s < 2 * kNumSMs && (d / (2 * s)) % gate::BK == 0) s *= 2;
    return s;
}

template <class TX>
void launch_gate_logits(const TX* x, const float* noise, const float* wg, float* logits,
                        int64_t T, int d, int E, int splits, cudaStream_t st) {
    dim3 grid((unsigned)ceil_div(T, gate::BT), (unsigned)ceil_div(E, gate::BE), (unsigned)splits);
    gate::logits_kernel<TX><<<grid, gate::NT, 0, st>>>(x, noise, wg, logits, T, d, E, d / splits);
    MOE_LAUNCH_CHECK();
}

template <class TIO>
void launch_gate_dx(int64_t T, int d, int E, int K, int cap_pad, const float* dL, const float* wg,
                    const float* noise, const TIO* dX, const int32_t* choice, const int32_t* pos,
                    const TIO* dy, bool residual_is_x, TIO* dx, TIO* dres, cudaStream_t st) {
    dim3 grid((unsigned)ceil_div(T, gate::BT), (unsigned)(d / gate::DJ));
    gate::dx_kernel<TIO><<<grid, gate::NT, 0, st>>>(T, d, E, K, cap_pad, dL, wg, noise, dX, choice,
                                                     pos, dy, residual_is_x, dx, dres);
    MOE_LAUNCH_CHECK();
}

template <class TX>
void launch_gate_dw(const TX* x, const float* noise, const float* dL, float* part, int64_t T,
                    int d, int E, int splits, cudaStream_t st) {
    const int64_t tps = round_up(ceil_div(T, splits), gate::BK);
    dim3 grid((unsigned)(d / gate::BT), (unsigned)ceil_div(E, gate::BE), (unsigned)splits);
    gate::dw_kernel<TX><<<grid, gate::NT, 0, st>>>(x, noise, dL, part, T, d, E, tps);
    MOE_LAUNCH_CHECK();
}

#define INST(T)                                                                                  \
    template void launch_gate_logits<T>(const T*, const float*, const float*, float*, int64_t,  \
                                        int, int, int, cudaStream_t);                            \
    template void launch_gate_dx<T>(int64_t, int, int, int, int, const float*, const float*,     \
                                    const float*, const T*, const int32_t*, const int32_t*,      \
                                    const T*, bool, T*, T*, cudaStream_t);                       \
    template void launch_gate_dw<T>(const T*, const float*, const float*, float*, int64_t, int,  \
                                    int, int, cudaStream_t);
INST(float)
INST(__nv_bfloat16)
#undef INST

}  // namespace moe
