// gate2.cu — second-generation gate GEMM kernels (fp32 FFMA, larger register
// tiles), used when d % 256 == 0 and E % 8 == 0, E <= 64 (every BASELINE
// config).  Semantics as gate.cu:
//   logits = (x * noise) Wg               routing.cpp:62-71
//   dx     = (dL Wg^T) * noise + sum_k dX[row_k] (+ dy)
//                                         ops.cpp:137-138, 223-228; routing.cpp:245-253, 337-342
#include "common.cuh"
#include "kernels.h"

namespace moe {
namespace gate2 {

constexpr int NT = 256;

// ---- logits: CTA = 128 tokens x 64 experts, thread = 8 tokens x 4 experts,
// K staged 32 at a time, split-K over blockIdx.z (partials summed in fixed
// order by the softmax kernel).
constexpr int LT = 128, LE = 64, LK = 32;

template <class TX>
__global__ void __launch_bounds__(NT)
logits_kernel(const TX* __restrict__ x, const float* __restrict__ noise,
              const float* __restrict__ wg, float* __restrict__ logits, int64_t T, int d, int E,
              int k_per_split) {
    pdl_wait();
    pdl_trigger();
    __shared__ __align__(16) float Xs[LK][LT + 4];
    __shared__ __align__(16) float Ws[LK][LE + 4];
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    const int64_t t0 = (int64_t)blockIdx.x * LT;
    const int e0 = blockIdx.y * LE;
    const int kb = blockIdx.z * k_per_split, ke = min(d, kb + k_per_split);
    logits += (int64_t)blockIdx.z * T * E;
    float acc[8][4] = {};
    const int xr = tid / 2, xh = tid % 2;  // staging: row, 16-k half
    for (int k0 = kb; k0 < ke; k0 += LK) {
        {
            float v[16];
            const int64_t t = t0 + xr;
            if (t < T) {
                const TX* xp = x + t * d + k0 + xh * 16;
                if constexpr (sizeof(TX) == 2) {
                    load_f<TX, 8>(xp, *reinterpret_cast<float(*)[8]>(v));
                    load_f<TX, 8>(xp + 8, *reinterpret_cast<float(*)[8]>(v + 8));
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) load_f<TX, 4>(xp + 4 * q, *reinterpret_cast<float(*)[4]>(v + 4 * q));
                }
                if (noise) {
                    const float* np_ = noise + t * d + k0 + xh * 16;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float4 nn = __ldg(reinterpret_cast<const float4*>(np_ + 4 * q));
                        v[4 * q] *= nn.x; v[4 * q + 1] *= nn.y; v[4 * q + 2] *= nn.z; v[4 * q + 3] *= nn.w;
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = 0.f;
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) Xs[xh * 16 + i][xr] = v[i];
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
        for (int k = 0; k < LK; ++k) {
            const float4 a0 = *reinterpret_cast<const float4*>(&Xs[k][ty * 8]);
            const float4 a1 = *reinterpret_cast<const float4*>(&Xs[k][ty * 8 + 4]);
            const float4 b = *reinterpret_cast<const float4*>(&Ws[k][tx * 4]);
            const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t t = t0 + ty * 8 + i;
        const int e = e0 + tx * 4;
        if (t < T && e < E)
            *reinterpret_cast<float4*>(logits + t * E + e) =
                make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    }
}

// ---- WgT = Wg^T ([E][d]) so the dx kernel stages contiguous rows.
__global__ void transpose_kernel(const float* __restrict__ wg, float* __restrict__ wgt, int d, int E) {
    pdl_wait();
    pdl_trigger();
    __shared__ float tile[32][33];
    const int j0 = blockIdx.x * 32, e0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int j = j0 + r, e = e0 + threadIdx.x;
        tile[r][threadIdx.x] = (j < d && e < E) ? wg[(int64_t)j * E + e] : 0.f;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int e = e0 + r, j = j0 + threadIdx.x;
        if (e < E && j < d) wgt[(int64_t)e * d + j] = tile[threadIdx.x][r];
    }
}

// ---- dx: CTA = 64 tokens x 256 columns, thread = 8 tokens x 8 columns;
// E staged in chunks of 16 rows of WgT.  With dxg_out set the kernel only
// writes dxg_out = (dL Wg^T) * noise in fp32 (the dispatch-backward gather is
// then done by dx_assemble); this variant runs on the side stream next to the
// expert weight-gradient GEMMs.
constexpr int DT = 64, DJ = 256, DE = 16, MAXE = 64;

template <class TIO>
__global__ void __launch_bounds__(NT)
dx_kernel(int64_t T, int d, int E, int K, int cap_pad, const float* __restrict__ dL,
          const float* __restrict__ wgt, const float* __restrict__ noise,
          const TIO* __restrict__ dX, const int32_t* __restrict__ choice,
          const int32_t* __restrict__ pos, const TIO* __restrict__ dy, bool residual_is_x,
          TIO* __restrict__ dx, TIO* __restrict__ dres, float* __restrict__ dxg_out) {
    pdl_wait();
    pdl_trigger();
    __shared__ __align__(16) float Ls[DT][MAXE + 1];
    __shared__ __align__(16) float Ws[DE][DJ + 4];
    __shared__ int64_t rows[DT][2];
    __shared__ int anyk[DT];
    const int tid = threadIdx.x;
    const int tx = tid % 32, ty = tid / 32;  // a warp shares its 8 tokens (broadcast reads)
    const int64_t t0 = (int64_t)blockIdx.x * DT;
    const int j0 = blockIdx.y * DJ;
    for (int i = tid; i < DT * E; i += NT) {
        const int tt = i / E, e = i % E;
        const int64_t t = t0 + tt;
        Ls[tt][e] = t < T ? dL[t * E + e] : 0.f;
    }
    if (tid < DT && !dxg_out) {
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
    float acc[8][8] = {};
    for (int ec = 0; ec < E; ec += DE) {
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int idx = tid + i * NT;  // 1024 float4 = 16 rows x 64
            const int er = idx / 64, c4 = idx % 64;
            float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
            if (ec + er < E) w = __ldg(reinterpret_cast<const float4*>(wgt + (int64_t)(ec + er) * d + j0 + c4 * 4));
            *reinterpret_cast<float4*>(&Ws[er][c4 * 4]) = w;
        }
        __syncthreads();
        const int ne = min(DE, E - ec);
        for (int ee = 0; ee < ne; ++ee) {
            float a[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = Ls[ty * 8 + i][ec + ee];
            const float4 b0 = *reinterpret_cast<const float4*>(&Ws[ee][tx * 8]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Ws[ee][tx * 8 + 4]);
            const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int q = 0; q < 8; ++q) acc[i][q] = fmaf(a[i], bv[q], acc[i][q]);
        }
    }
    const int j = j0 + tx * 8;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int tt = ty * 8 + i;
        const int64_t t = t0 + tt;
        if (t >= T) continue;
        float v[8];
        if (noise) {
            const float4 n0 = __ldg(reinterpret_cast<const float4*>(noise + t * d + j));
            const float4 n1 = __ldg(reinterpret_cast<const float4*>(noise + t * d + j + 4));
            const float nv[8] = {n0.x, n0.y, n0.z, n0.w, n1.x, n1.y, n1.z, n1.w};
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = acc[i][q] * nv[q];
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = acc[i][q];
        }
        if (dxg_out) {
            *reinterpret_cast<float4*>(dxg_out + t * d + j) = make_float4(v[0], v[1], v[2], v[3]);
            *reinterpret_cast<float4*>(dxg_out + t * d + j + 4) = make_float4(v[4], v[5], v[6], v[7]);
            continue;
        }
        #pragma unroll
        for (int k = 0; k < 2; ++k) {  // K <= 2
            if (k >= K) break;
            const int64_t r = rows[tt][k];
            if (r < 0) continue;
            float g[8];
            if constexpr (sizeof(TIO) == 2) {
                load_f<TIO, 8>(dX + r * d + j, g);
            } else {
                load_f<TIO, 4>(dX + r * d + j, *reinterpret_cast<float(*)[4]>(g));
                load_f<TIO, 4>(dX + r * d + j + 4, *reinterpret_cast<float(*)[4]>(g + 4));
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] += g[q];
        }
        auto st8 = [&](TIO* p, float (&s)[8]) {
            if constexpr (sizeof(TIO) == 2) {
                store_f<TIO, 8>(p, s);
            } else {
                store_f<TIO, 4>(p, *reinterpret_cast<float(*)[4]>(s));
                store_f<TIO, 4>(p + 4, *reinterpret_cast<float(*)[4]>(s + 4));
            }
        };
        if (!anyk[tt]) {
            float g[8];
            if constexpr (sizeof(TIO) == 2) {
                load_f<TIO, 8>(dy + t * d + j, g);
            } else {
                load_f<TIO, 4>(dy + t * d + j, *reinterpret_cast<float(*)[4]>(g));
                load_f<TIO, 4>(dy + t * d + j + 4, *reinterpret_cast<float(*)[4]>(g + 4));
            }
            if (residual_is_x) {
#pragma unroll
                for (int q = 0; q < 8; ++q) v[q] += g[q];
            } else if (dres) {
                st8(dres + t * d + j, g);
            }
        } else if (!residual_is_x && dres) {
            float z[8] = {};
            st8(dres + t * d + j, z);
        }
        st8(dx + t * d + j, v);
    }
}

}  // namespace gate2

bool gate2_ok(int d, int E) { return d % gate2::DJ == 0 && E % 8 == 0 && E <= gate2::MAXE; }

template <class TX>
void launch_gate2_logits(const TX* x, const float* noise, const float* wg, float* logits, int64_t T,
                         int d, int E, int splits, cudaStream_t st) {
    dim3 grid((unsigned)ceil_div(T, gate2::LT), (unsigned)ceil_div(E, gate2::LE), (unsigned)splits);
    launch_pdl(gate2::logits_kernel<TX>, dim3(grid), dim3(gate2::NT), 0, st, x, noise, wg, logits, T, d, E, d / splits);
}

void launch_gate2_transpose(const float* wg, float* wgt, int d, int E, cudaStream_t st) {
    dim3 grid((unsigned)ceil_div(d, 32), (unsigned)ceil_div(E, 32));
    launch_pdl(gate2::transpose_kernel, dim3(grid), dim3(dim3(32, 8)), 0, st, wg, wgt, d, E);
}

template <class TIO>
void launch_gate2_dx(int64_t T, int d, int E, int K, int cap_pad, const float* dL, const float* wgt,
                     const float* noise, const TIO* dX, const int32_t* choice, const int32_t* pos,
                     const TIO* dy, bool residual_is_x, TIO* dx, TIO* dres, cudaStream_t st) {
    dim3 grid((unsigned)ceil_div(T, gate2::DT), (unsigned)(d / gate2::DJ));
    launch_pdl(gate2::dx_kernel<TIO>, dim3(grid), dim3(gate2::NT), 0, st, T, d, E, K, cap_pad, dL, wgt, noise, dX, choice,
                                                       pos, dy, residual_is_x, dx, dres, nullptr);
}

void launch_gate2_dxg(int64_t T, int d, int E, const float* dL, const float* wgt, const float* noise,
                      float* dxg, cudaStream_t st) {
    dim3 grid((unsigned)ceil_div(T, gate2::DT), (unsigned)(d / gate2::DJ));
    launch_pdl(gate2::dx_kernel<float>, dim3(grid), dim3(gate2::NT), 0, st, T, d, E, 1, 0, dL, wgt, noise, nullptr, nullptr,
                                                         nullptr, nullptr, false, nullptr, nullptr, dxg);
}

int gate2_logit_splits(int64_t T, int d, int E) {
    const int64_t ctas = ceil_div(T, gate2::LT) * ceil_div(E, gate2::LE);
    int s = 1;
    while (s < kMaxGateSplits && ctas * s < 2 * kNumSMs && (d / (2 * s)) % gate2::LK == 0) s *= 2;
    return s;
}

#define INST(T)                                                                                     \
    template void launch_gate2_logits<T>(const T*, const float*, const float*, float*, int64_t,    \
                                         int, int, int, cudaStream_t);                              \
    template void launch_gate2_dx<T>(int64_t, int, int, int, int, const float*, const float*,       \
                                     const float*, const T*, const int32_t*, const int32_t*,        \
                                     const T*, bool, T*, T*, cudaStream_t);
INST(float)
INST(__nv_bfloat16)
#undef INST

}  // namespace moe
