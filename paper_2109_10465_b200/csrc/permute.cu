// permute.cu — dispatch / combine permutation kernels and their backwards.
//
// Reference semantics (relative to /root/reference/proj/core/src):
//   dispatch  routing.cpp:208-256   buf[e*cap + slot] = x[t]; bwd dx[t] += dbuf[row]
//   combine   routing.cpp:258-346   y[t] = sum_k w_k O[row_k] (or residual if none kept);
//                                   bwd dO[row] += w dy[t]; dw = <dy, O[row]>
//   weights   routing.cpp:408-417   top-1 w = E * p; top-2 w_k = p_k / (p_0 + p_1)
//
// Every kernel is a row gather with 16-byte vector loads/stores, one warp per
// row, so each output row is written exactly once (no atomics, deterministic).
// The fused layer uses a compact internal row index e*cap_pad + pos (pos ==
// slot except in grouped mode) whose occupied rows are dense per expert.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace moe {

constexpr int kRowWarps = 8;

// buf row r of expert e: src = row_src[r] if pos < kept[e]; zero-filled for
// pos in [kept[e], roundup(kept[e], 128)) so the tensor-core tiles never read
// stale rows; rows beyond that are never read.
template <class TIO, int V>
__global__ void __launch_bounds__(kRowWarps * 32)
dispatch_gather_kernel(const TIO* __restrict__ x, int64_t d, int E, int K, int cap_pad,
                       const int32_t* __restrict__ row_src, const int32_t* __restrict__ kept,
                       TIO* __restrict__ buf, RowDst rd) {
    pdl_wait();
    pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * kRowWarps + warp;
    if (r >= (int64_t)E * cap_pad) return;
    const int e = (int)(r / cap_pad);
    const int p = (int)(r % cap_pad);
    const int n = kept[e];
    // expert parallelism: the row goes straight to its expert owner's receive
    // buffer (NVLink store; rd.p[o] already points at this rank's slot there)
    TIO* dst = rd.ep > 1 ? static_cast<TIO*>(rd.p[e / rd.El]) + ((int64_t)(e % rd.El) * cap_pad + p) * d
                         : buf + r * d;
    if (p < n) {
        const int64_t t = row_src[r] / K;
        const TIO* src = x + t * d;
        if constexpr (V * sizeof(TIO) == 16) {
            // kU 16-byte loads in flight per lane before the stores
            constexpr int kU = 8;
            for (int64_t j0 = (int64_t)lane * V; j0 < d; j0 += 32 * V * kU) {
                uint4 v[kU];
#pragma unroll
                for (int u = 0; u < kU; ++u)
                    if (j0 + u * 32 * V < d) v[u] = __ldg(reinterpret_cast<const uint4*>(src + j0 + u * 32 * V));
#pragma unroll
                for (int u = 0; u < kU; ++u)
                    if (j0 + u * 32 * V < d) *reinterpret_cast<uint4*>(dst + j0 + u * 32 * V) = v[u];
            }
        } else {
            for (int64_t j = (int64_t)lane * V; j < d; j += 32 * V) copy_vec<TIO, V>(dst + j, src + j);
        }
    } else if (p < round_up_dev(n, kRowAlign)) {
        for (int64_t j = (int64_t)lane * V; j < d; j += 32 * V) zero_vec<TIO, V>(dst + j);
    }
}

template <class TIO>
void launch_dispatch_gather(const TIO* x, int64_t d, int E, int K, int cap_pad,
                            const int32_t* row_src, const int32_t* kept, TIO* buf,
                            uint32_t* flags, cudaStream_t st, const RowDst* rd) {
    (void)flags;
    const int64_t rows = (int64_t)E * cap_pad;
    const unsigned grid = (unsigned)ceil_div(rows, kRowWarps);
    RowDst r0{};
    const RowDst& rdv = rd ? *rd : r0;
    if (vec_width<TIO>(d) > 1)
        launch_pdl(dispatch_gather_kernel<TIO, 16 / sizeof(TIO)>, dim3(grid), dim3(kRowWarps * 32), 0, st,
            x, d, E, K, cap_pad, row_src, kept, buf, rdv);
    else
        launch_pdl(dispatch_gather_kernel<TIO, 1>, dim3(grid), dim3(kRowWarps * 32), 0, st, x, d, E, K, cap_pad,
                   row_src, kept, buf, rdv);
}

// y[t] = sum_{k kept} w[t*K+k] * O[row_k]  (accumulated from 0 in k order,
// routing.cpp:279-292), else the residual row.
template <class TIO, int V>
__global__ void __launch_bounds__(kRowWarps * 32)
combine_kernel(const TIO* __restrict__ O, int64_t T, int64_t d, int K, int cap_pad,
               const int32_t* __restrict__ choice, const int32_t* __restrict__ pos,
               const float* __restrict__ w, const TIO* __restrict__ residual, TIO* __restrict__ y,
               uint32_t* __restrict__ flags) {
    pdl_wait();
    pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t = (int64_t)blockIdx.x * kRowWarps + warp;
    if (t >= T) return;
    int64_t rows[2] = {-1, -1};
    float wk[2] = {0.f, 0.f};
    bool any = false;
#pragma unroll
    for (int k = 0; k < 2; ++k) {  // K <= 2; unrolled so rows / wk stay in registers
        if (k >= K) break;
        const int32_t p = pos[t * K + k];
        if (p >= 0) {
            rows[k] = (int64_t)choice[t * K + k] * cap_pad + p;
            wk[k] = w[t * K + k];
            any = true;
        }
    }
    bool bad = false;
    for (int64_t j = (int64_t)lane * V; j < d; j += 32 * V) {
        float acc[V];
        if (any) {
#pragma unroll
            for (int q = 0; q < V; ++q) acc[q] = 0.f;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                if (k >= K || rows[k] < 0) continue;
                float o[V];
                load_f<TIO, V>(O + rows[k] * d + j, o);
#pragma unroll
                for (int q = 0; q < V; ++q) acc[q] = fmaf(wk[k], o[q], acc[q]);
            }
        } else {
            load_f<TIO, V>(residual + t * d + j, acc);
        }
#pragma unroll
        for (int q = 0; q < V; ++q) bad |= !finite_f(acc[q]);
        store_f<TIO, V>(y + t * d + j, acc);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, MOE_FLAG_NONFINITE_DEV);
}

template <class TIO>
void launch_combine(const TIO* O, int64_t T, int64_t d, int E, int K, int cap_pad,
                    const int32_t* choice, const int32_t* pos, const float* w,
                    const TIO* residual, TIO* y, uint32_t* flags, cudaStream_t st) {
    (void)E;
    const unsigned grid = (unsigned)ceil_div(T, kRowWarps);
    if (vec_width<TIO>(d) > 1)
        launch_pdl(combine_kernel<TIO, 16 / sizeof(TIO)>, dim3(grid), dim3(kRowWarps * 32), 0, st, 
            O, T, d, K, cap_pad, choice, pos, w, residual, y, flags);
    else
        launch_pdl(combine_kernel<TIO, 1>, dim3(grid), dim3(kRowWarps * 32), 0, st, O, T, d, K, cap_pad, choice, pos,
                                                                w, residual, y, flags);
}

// dO[r] = w[src] * dy[t(src)] for occupied rows; zero tail up to 128 rows.
template <class TIO, int V>
__global__ void __launch_bounds__(kRowWarps * 32)
combine_bwd_gather_kernel(const TIO* __restrict__ dy, int64_t d, int K, int cap_pad,
                          const int32_t* __restrict__ row_src, const int32_t* __restrict__ kept,
                          const float* __restrict__ w, TIO* __restrict__ dO, int64_t rows) {
    pdl_wait();
    pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * kRowWarps + warp;
    if (r >= rows) return;
    const int e = (int)(r / cap_pad);
    const int p = (int)(r % cap_pad);
    const int n = kept[e];
    TIO* dst = dO + r * d;
    if (p < n) {
        const int32_t src = row_src[r];
        const float wv = w[src];
        const TIO* s = dy + (int64_t)(src / K) * d;
        for (int64_t j = (int64_t)lane * V; j < d; j += 32 * V) {
            float v[V];
            load_f<TIO, V>(s + j, v);
#pragma unroll
            for (int q = 0; q < V; ++q) v[q] *= wv;
            store_f<TIO, V>(dst + j, v);
        }
    } else if (p < round_up_dev(n, kRowAlign)) {
        for (int64_t j = (int64_t)lane * V; j < d; j += 32 * V) zero_vec<TIO, V>(dst + j);
    }
}

template <class TIO>
void launch_combine_bwd_gather(const TIO* dy, int64_t d, int E, int K, int cap_pad,
                               const int32_t* row_src, const int32_t* kept, const float* w,
                               TIO* dO, cudaStream_t st) {
    const int64_t rows = (int64_t)E * cap_pad;
    const unsigned grid = (unsigned)ceil_div(rows, kRowWarps);
    if (vec_width<TIO>(d) > 1)
        launch_pdl(combine_bwd_gather_kernel<TIO, 16 / sizeof(TIO)>, dim3(grid), dim3(kRowWarps * 32), 0, st, 
            dy, d, K, cap_pad, row_src, kept, w, dO, rows);
    else
        launch_pdl(combine_bwd_gather_kernel<TIO, 1>, dim3(grid), dim3(kRowWarps * 32), 0, st, dy, d, K, cap_pad,
                                                                           row_src, kept, w, dO, rows);
}

// dx[t] = dxg[t] * noise[t] + sum_{k kept} dX[row_k] (+ dy[t] if no route kept
// and the residual is x).  Mirrors the three tape contributions to dx:
// jitter mul bwd (ops.cpp:223-228), dispatch bwd (routing.cpp:245-253) and
// the combine residual branch (routing.cpp:337-342).
template <class TIO, int V>
__global__ void __launch_bounds__(kRowWarps * 32)
dx_assemble_kernel(int64_t T, int64_t d, int K, int cap_pad, const float* __restrict__ dxg,
                   const float* __restrict__ noise, const TIO* __restrict__ dX,
                   const int32_t* __restrict__ choice, const int32_t* __restrict__ pos,
                   const TIO* __restrict__ dy, bool residual_is_x, TIO* __restrict__ dx,
                   TIO* __restrict__ dres) {
    pdl_wait();
    pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t = (int64_t)blockIdx.x * kRowWarps + warp;
    if (t >= T) return;
    int64_t rows[2] = {-1, -1};
    bool any = false;
    #pragma unroll
    for (int k = 0; k < 2; ++k) {  // K <= 2
        if (k >= K) break;
        const int32_t p = pos[t * K + k];
        if (p >= 0) {
            rows[k] = (int64_t)choice[t * K + k] * cap_pad + p;
            any = true;
        }
    }
    for (int64_t j = (int64_t)lane * V; j < d; j += 32 * V) {
        float acc[V];
#pragma unroll
        for (int q = 0; q < V; ++q) acc[q] = 0.f;
        #pragma unroll
        for (int k = 0; k < 2; ++k) {  // K <= 2
            if (k >= K) break;
            if (rows[k] < 0) continue;
            float v[V];
            load_f<TIO, V>(dX + rows[k] * d + j, v);
#pragma unroll
            for (int q = 0; q < V; ++q) acc[q] += v[q];
        }
        {
            float g[V];
            if constexpr (V % 4 == 0) {
#pragma unroll
                for (int q = 0; q < V; q += 4) {
                    const float4 u = __ldg(reinterpret_cast<const float4*>(dxg + t * d + j + q));
                    g[q] = u.x; g[q + 1] = u.y; g[q + 2] = u.z; g[q + 3] = u.w;
                }
            } else {
#pragma unroll
                for (int q = 0; q < V; ++q) g[q] = dxg[t * d + j + q];
            }
#pragma unroll
            for (int q = 0; q < V; ++q) {
                const float nz = noise ? noise[t * d + j + q] : 1.f;
                acc[q] = fmaf(g[q], nz, acc[q]);
            }
        }
        if (!any) {
            float g[V];
            load_f<TIO, V>(dy + t * d + j, g);
            if (residual_is_x) {
#pragma unroll
                for (int q = 0; q < V; ++q) acc[q] += g[q];
            } else if (dres) {
                store_f<TIO, V>(dres + t * d + j, g);
            }
        } else if (!residual_is_x && dres) {
            zero_vec<TIO, V>(dres + t * d + j);
        }
        store_f<TIO, V>(dx + t * d + j, acc);
    }
}

template <class TIO>
void launch_dx_assemble(int64_t T, int64_t d, int E, int K, int cap_pad, const float* dxg,
                        const float* noise, const TIO* dX, const int32_t* choice,
                        const int32_t* pos, const TIO* dy, bool residual_is_x, TIO* dx,
                        TIO* dres, cudaStream_t st) {
    (void)E;
    const unsigned grid = (unsigned)ceil_div(T, kRowWarps);
    if (vec_width<TIO>(d) > 1)
        launch_pdl(dx_assemble_kernel<TIO, 16 / sizeof(TIO)>, dim3(grid), dim3(kRowWarps * 32), 0, st, 
            T, d, K, cap_pad, dxg, noise, dX, choice, pos, dy, residual_is_x, dx, dres);
    else
        launch_pdl(dx_assemble_kernel<TIO, 1>, dim3(grid), dim3(kRowWarps * 32), 0, st, 
            T, d, K, cap_pad, dxg, noise, dX, choice, pos, dy, residual_is_x, dx, dres);
}

// Utilization + drop statistics of one routing decision, accumulated into
// caller-owned int64 counters (integer adds: exact and order-free):
//   util[e]  += #{t : first choice of t is e}            surgery.cpp:113-118
//   hist[b]  += #{dropped routes of tokens t with min(7, 8t/T) = b}
//   hist[8]  += #dropped routes, hist[9] += T*K           trainer.cpp:15-29
__global__ void decision_stats_kernel(int64_t T, int E, int K, const int32_t* __restrict__ choice,
                                      const int32_t* __restrict__ pos,
                                      unsigned long long* __restrict__ util,
                                      unsigned long long* __restrict__ hist) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ unsigned int s_cnt[];  // [E] + [9]
    for (int i = threadIdx.x; i < E + 9; i += blockDim.x) s_cnt[i] = 0;
    __syncthreads();
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int c0 = choice[t * K];
        if (c0 >= 0 && c0 < E) atomicAdd(&s_cnt[c0], 1u);
        #pragma unroll
        for (int k = 0; k < 2; ++k) {  // K <= 2
            if (k >= K) break;
            if (pos[t * K + k] >= 0) continue;
            const int64_t tb = t * 8 / (T > 1 ? T : 1);
            const int b = tb < 7 ? (int)tb : 7;
            atomicAdd(&s_cnt[E + b], 1u);
            atomicAdd(&s_cnt[E + 8], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < E + 9; i += blockDim.x) {
        const unsigned long long v = s_cnt[i];
        if (v == 0) continue;
        if (i < E) atomicAdd(&util[i], v);
        else atomicAdd(&hist[i - E], v);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&hist[9], (unsigned long long)(T * K));
}

void launch_decision_stats(int64_t T, int E, int K, const int32_t* choice, const int32_t* pos,
                           int64_t* util, int64_t* hist, cudaStream_t st) {
    const int blocks = (int)std::min<int64_t>(kNumSMs, ceil_div(T, (int64_t)256));
    launch_pdl(decision_stats_kernel, dim3(blocks), dim3(256), sizeof(unsigned int) * (E + 9), st, 
        T, E, K, choice, pos, reinterpret_cast<unsigned long long*>(util),
        reinterpret_cast<unsigned long long*>(hist));
}

__global__ void combine_weights_kernel(int64_t T, int E, int K, const float* __restrict__ gp,
                                       float* __restrict__ w) {
    pdl_wait();
    pdl_trigger();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    if (K == 1) {
        w[t] = gp[t] * (float)E;  // scale(gate_prob, E), routing.cpp:408-411
    } else {
        const float p0 = gp[2 * t], p1 = gp[2 * t + 1];
        const float s = p0 + p1;  // add + div_elem, routing.cpp:412-416
        w[2 * t] = p0 / s;
        w[2 * t + 1] = p1 / s;
    }
}

void launch_combine_weights(int64_t T, int E, int K, const float* gate_prob, float* w,
                            cudaStream_t st) {
    launch_pdl(combine_weights_kernel, dim3((unsigned)ceil_div(T, 256)), dim3(256), 0, st, T, E, K, gate_prob, w);
}

// db[g][n] = sum_{r, i < count(r,g)} src[(r*El+g)*cap_pad + i][n], fixed order.
// One CTA per SM at most (grid-stride over (group, 128-column block) items):
// the kernel runs on the side stream next to persistent GEMMs and must never
// take the registers / warp slots a GEMM CTA needs.  4 row groups per item
// (fixed strided order), combined in fixed order through shared memory.
constexpr int kColsumRG = 4;
template <class TIO>
__global__ void __launch_bounds__(128 * kColsumRG)
colsum_groups_kernel(const TIO* __restrict__ src, int64_t N, int ep, int El, int cap_pad,
                     const int32_t* __restrict__ counts, float* __restrict__ db) {
    pdl_wait();
    pdl_trigger();
    __shared__ float part[kColsumRG][128];
    const int c = threadIdx.x & 127, rg = threadIdx.x >> 7;
    const int64_t nblk = (N + 127) / 128;
    for (int64_t item = blockIdx.x; item < nblk * El; item += gridDim.x) {
        const int g = static_cast<int>(item / nblk);
        const int64_t n = (item % nblk) * 128 + c;
        float acc = 0.f;
        if (n < N) {
            for (int r = 0; r < ep; ++r) {
                const int seg = r * El + g;
                const int cnt = counts[seg];
                const TIO* base = src + (int64_t)seg * cap_pad * N + n;
                for (int i = rg; i < cnt; i += kColsumRG) acc += to_f(base[(int64_t)i * N]);
            }
        }
        part[rg][c] = acc;
        __syncthreads();
        if (rg == 0 && n < N) {
            float t = part[0][c];
#pragma unroll
            for (int q = 1; q < kColsumRG; ++q) t += part[q][c];
            db[(int64_t)g * N + n] = t;
        }
        __syncthreads();
    }
}

template <class TIO>
void launch_colsum_groups(const TIO* src, int64_t N, int ep, int El, int cap_pad,
                          const int32_t* counts, float* db, cudaStream_t st) {
    const int64_t items = ceil_div(N, (int64_t)128) * El;
    launch_pdl(colsum_groups_kernel<TIO>, dim3((unsigned)std::min<int64_t>(items, kNumSMs)), dim3(128 * kColsumRG), 0, st, 
        src, N, ep, El, cap_pad, counts, db);
}

__global__ void colsum_parts_kernel(const float* __restrict__ part, int64_t N, int ep, int El,
                                    int cap_pad, const int32_t* __restrict__ counts,
                                    float* __restrict__ db) {
    pdl_wait();
    pdl_trigger();
    const int g = blockIdx.y;
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    float acc = 0.f;
    for (int r = 0; r < ep; ++r) {
        const int seg = r * El + g;
        // 32-row blocks of the 128-row tiles the GEMM computed for this segment
        const int nblk = 4 * ((counts[seg] + 127) / 128);
        const float* base = part + ((int64_t)seg * cap_pad / 32) * N + n;
        for (int b = 0; b < nblk; ++b) acc += base[(int64_t)b * N];
    }
    db[(int64_t)g * N + n] = acc;
}

void launch_colsum_parts(const float* part, int64_t N, int ep, int El, int cap_pad,
                         const int32_t* counts, float* db, cudaStream_t st) {
    dim3 grid((unsigned)ceil_div(N, 128), El);
    launch_pdl(colsum_parts_kernel, dim3(grid), dim3(128), 0, st, part, N, ep, El, cap_pad, counts, db);
}

__global__ void convert_f64_kernel(const double* __restrict__ src, int64_t n, bool bf16, void* dst) {
    pdl_wait();
    pdl_trigger();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (bf16) static_cast<__nv_bfloat16*>(dst)[i] = __double2bfloat16(src[i]);
        else static_cast<float*>(dst)[i] = __double2float_rn(src[i]);
    }
}

void launch_convert_f64(const double* src, int64_t n, bool bf16, void* dst, cudaStream_t st) {
    if (n <= 0) return;
    launch_pdl(convert_f64_kernel, dim3((unsigned)std::min<int64_t>(8 * kNumSMs, ceil_div(n, (int64_t)256))), dim3(256), 0, st, 
        src, n, bf16, dst);
}

// ---- reference-layout per-stage kernels ------------------------------------
template <class TIO>
__global__ void dispatch_ref_kernel(const TIO* __restrict__ x, int64_t T, int64_t d, int K,
                                    int cap, const int32_t* __restrict__ eid,
                                    const int32_t* __restrict__ slot, TIO* __restrict__ buf,
                                    uint8_t* __restrict__ occ) {
    pdl_wait();
    pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * kRowWarps + warp;  // route index
    if (i >= T * K) return;
    const int32_t s = slot[i];
    if (s < 0) return;
    const int64_t row = (int64_t)eid[i] * cap + s;
    const int64_t t = i / K;
    for (int64_t j = lane; j < d; j += 32) buf[row * d + j] = x[t * d + j];
    if (lane == 0 && occ) occ[row] = 1;
}

template <class TIO>
void launch_dispatch_ref(const TIO* x, int64_t T, int64_t d, int E, int K, int cap,
                         const int32_t* expert_id, const int32_t* slot, TIO* buf, uint8_t* occ,
                         cudaStream_t st) {
    MOE_CUDA_CHECK(cudaMemsetAsync(buf, 0, sizeof(TIO) * (size_t)E * cap * d, st));
    if (occ) MOE_CUDA_CHECK(cudaMemsetAsync(occ, 0, (size_t)E * cap, st));
    if (T * K == 0) return;
    launch_pdl(dispatch_ref_kernel<TIO>, dim3((unsigned)ceil_div(T * K, kRowWarps)), dim3(kRowWarps * 32), 0, st, 
        x, T, d, K, cap, expert_id, slot, buf, occ);
}

template <class TIO>
__global__ void combine_ref_kernel(const TIO* __restrict__ O, int64_t T, int64_t d, int K,
                                   int cap, const int32_t* __restrict__ eid,
                                   const int32_t* __restrict__ slot, const float* __restrict__ w,
                                   const TIO* __restrict__ residual, TIO* __restrict__ y) {
    pdl_wait();
    pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t = (int64_t)blockIdx.x * kRowWarps + warp;
    if (t >= T) return;
    bool any = false;
    for (int k = 0; k < K; ++k) any |= slot[t * K + k] >= 0;
    for (int64_t j = lane; j < d; j += 32) {
        float acc = 0.f;
        if (any) {
            #pragma unroll
            for (int k = 0; k < 2; ++k) {  // K <= 2
                if (k >= K) break;
                const int32_t s = slot[t * K + k];
                if (s < 0) continue;
                acc = fmaf(w[(int64_t)k * T + t], to_f(O[((int64_t)eid[t * K + k] * cap + s) * d + j]), acc);
            }
        } else {
            acc = to_f(residual[t * d + j]);
        }
        y[t * d + j] = from_f<TIO>(acc);
    }
}

template <class TIO>
void launch_combine_ref(const TIO* O, int64_t T, int64_t d, int E, int K, int cap,
                        const int32_t* expert_id, const int32_t* slot, const float* w,
                        const TIO* residual, TIO* y, cudaStream_t st) {
    (void)E;
    launch_pdl(combine_ref_kernel<TIO>, dim3((unsigned)ceil_div(T, kRowWarps)), dim3(kRowWarps * 32), 0, st, 
        O, T, d, K, cap, expert_id, slot, w, residual, y);
}

__global__ void check_finite_kernel(const float* __restrict__ p, int64_t n, uint32_t* flags) {
    pdl_wait();
    pdl_trigger();
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        bad |= !finite_f(p[i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, MOE_FLAG_NONFINITE_DEV);
}

void launch_check_finite_f32(const float* p, int64_t n, uint32_t* flags, cudaStream_t st) {
    if (n <= 0) return;
    launch_pdl(check_finite_kernel, dim3((unsigned)std::min<int64_t>(ceil_div(n, 256), 4 * kNumSMs)), dim3(256), 0, st, 
        p, n, flags);
}

#define INST(T)                                                                                  \
    template void launch_dispatch_gather<T>(const T*, int64_t, int, int, int, const int32_t*,   \
                                            const int32_t*, T*, uint32_t*, cudaStream_t,        \
                                            const RowDst*);                                      \
    template void launch_combine<T>(const T*, int64_t, int64_t, int, int, int, const int32_t*,   \
                                    const int32_t*, const float*, const T*, T*, uint32_t*,       \
                                    cudaStream_t);                                               \
    template void launch_combine_bwd_gather<T>(const T*, int64_t, int, int, int, const int32_t*, \
                                               const int32_t*, const float*, T*, cudaStream_t);  \
    template void launch_dx_assemble<T>(int64_t, int64_t, int, int, int, const float*,           \
                                        const float*, const T*, const int32_t*, const int32_t*,  \
                                        const T*, bool, T*, T*, cudaStream_t);                   \
    template void launch_colsum_groups<T>(const T*, int64_t, int, int, int, const int32_t*,      \
                                          float*, cudaStream_t);                                 \
    template void launch_dispatch_ref<T>(const T*, int64_t, int64_t, int, int, int,              \
                                         const int32_t*, const int32_t*, T*, uint8_t*,           \
                                         cudaStream_t);                                          \
    template void launch_combine_ref<T>(const T*, int64_t, int64_t, int, int, int,               \
                                        const int32_t*, const int32_t*, const float*, const T*,  \
                                        T*, cudaStream_t);
INST(float)
INST(__nv_bfloat16)
#undef INST

}  // namespace moe

namespace moe {

// Multi-destination copy for the expert-parallel exchange: up to kMaxCopies
// (src, dst, bytes) jobs, dst typically a peer GPU's buffer mapped over
// NVLink (CUDA IPC).  16-byte vectors, 4 in flight per thread, grid-stride
// over the concatenation of all jobs.
// Each job (one destination slice) gets a contiguous range of CTAs in
// proportion to its size; a CTA streams 16-byte vectors, 8 per thread in
// flight, from local HBM to the (local or NVLink peer) destination.
__global__ void __launch_bounds__(256) peer_copy_kernel(PeerCopyJobs jobs, int ctas_per_job) {
    pdl_wait();
    pdl_trigger();
    const int j = blockIdx.x / ctas_per_job;
    if (j >= jobs.n) return;
    const int64_t nv = jobs.bytes[j] >> 4;
    const uint4* __restrict__ src = reinterpret_cast<const uint4*>(jobs.src[j]);
    uint4* __restrict__ dst = reinterpret_cast<uint4*>(jobs.dst[j]);
    const int64_t stride = (int64_t)ctas_per_job * blockDim.x;
    constexpr int U = 8;
    for (int64_t v = (int64_t)(blockIdx.x % ctas_per_job) * blockDim.x + threadIdx.x; v < nv; v += U * stride) {
        uint4 buf[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (v + u * stride < nv) buf[u] = __ldg(src + v + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (v + u * stride < nv) dst[v + u * stride] = buf[u];
    }
}

void launch_peer_copy(const PeerCopyJobs& jobs, cudaStream_t st) {
    int64_t maxv = 0;
    for (int j = 0; j < jobs.n; ++j) {
        if ((jobs.bytes[j] & 15) || (reinterpret_cast<uintptr_t>(jobs.src[j]) & 15) ||
            (reinterpret_cast<uintptr_t>(jobs.dst[j]) & 15))
            throw Status(1, "peer copy: 16-byte alignment required");
        maxv = std::max<int64_t>(maxv, jobs.bytes[j] >> 4);
    }
    if (maxv == 0 || jobs.n == 0) return;
    const int per = (int)std::max<int64_t>(1, std::min<int64_t>(4 * kNumSMs / jobs.n, ceil_div(maxv, (int64_t)256 * 8)));
    launch_pdl(peer_copy_kernel, dim3(per * jobs.n), dim3(256), 0, st, jobs, per);
}

// out[i] = sum_r src[r][i] over the ranks' (NVLink-mapped) copies, in rank
// order: every rank computes the identical fp32 sum.
struct RankSrcs {
    const float* p[8];
};
__global__ void sum_ranks_kernel(RankSrcs s, int ep, int64_t n, float* __restrict__ out) {
    pdl_wait();
    pdl_trigger();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 acc = reinterpret_cast<const float4*>(s.p[0])[i];
        for (int r = 1; r < ep; ++r) {
            const float4 v = reinterpret_cast<const float4*>(s.p[r])[i];
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        reinterpret_cast<float4*>(out)[i] = acc;
    }
}

void launch_sum_ranks(const float* const* srcs, int ep, int64_t n, float* out, cudaStream_t st) {
    if (n % 4) throw Status(1, "sum_ranks: element count must be a multiple of 4");
    RankSrcs s{};
    for (int r = 0; r < ep; ++r) s.p[r] = srcs[r];
    launch_pdl(sum_ranks_kernel, dim3((unsigned)std::min<int64_t>(2 * kNumSMs, ceil_div(n / 4, (int64_t)256))), dim3(256), 0, st, 
        s, ep, n, out);
}

// Device-side barrier over NVLink peer memory for the IPC exchanges: every
// rank stores `epoch` into its slot of every peer's flag array (release,
// system scope, after a system fence so the preceding copy kernel's peer
// stores are ordered before it), then waits until every slot of its own array
// has reached `epoch` (acquire).  One warp; a ~30 s clock budget traps
// instead of hanging forever if a peer never arrives.
//
// With a ShapeCheck the barrier also carries each rank's token count: rank r
// stores T_r into slot kShapeSlot + r of every peer's array before its epoch
// (same release), and after the acquire compares every rank's T with its own.
// Unequal per-rank T is the reference's UniformShapeError
// (parallel.cpp:245-253): the flag latches MOE_FLAG_UNIFORM_SHAPE and the
// received per-expert counts are zeroed so no expert GEMM touches rows laid
// out for another rank's capacity.
constexpr int kShapeSlot = 8;
__global__ void ipc_barrier_kernel(PeerFlags peers, const unsigned long long* mine, int rank, int ep,
                                   unsigned long long epoch, ShapeCheck sc) {
    pdl_wait();
    pdl_trigger();
    const int i = threadIdx.x;
    bool bad = false;
    if (i < ep) {
        if (sc.tokens >= 0)
            asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(peers.f[i] + kShapeSlot + rank),
                         "l"((unsigned long long)sc.tokens) : "memory");
        __threadfence_system();
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peers.f[i] + rank), "l"(epoch) : "memory");
        unsigned long long v;
        const long long t0 = clock64();
        do {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine + i) : "memory");
            if (clock64() - t0 > (1LL << 36)) __trap();
        } while (v < epoch);
        if (sc.tokens >= 0) {
            unsigned long long t;
            asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(t) : "l"(mine + kShapeSlot + i) : "memory");
            bad = t != (unsigned long long)sc.tokens;
        }
    }
    if (__any_sync(0xffffffffu, bad)) {
        for (int c = i; c < sc.ncounts; c += 32) sc.counts[c] = 0;
        if (i == 0) atomicOr(sc.flags, MOE_FLAG_UNIFORM_SHAPE_DEV);
    }
}

void launch_ipc_barrier(const PeerFlags& peers, const unsigned long long* mine, int rank, int ep,
                        unsigned long long epoch, cudaStream_t st, const ShapeCheck* sc) {
    ShapeCheck none{};
    none.tokens = -1;
    launch_pdl(ipc_barrier_kernel, dim3(1), dim3(32), 0, st, peers, mine, rank, ep, epoch, sc ? *sc : none);
}

// NCCL transport: `all_t` holds every rank's token count (all-gathered).
__global__ void ep_shape_check_kernel(const long long* all_t, int ep, ShapeCheck sc) {
    pdl_wait();
    pdl_trigger();
    const int i = threadIdx.x;
    const bool bad = i < ep && all_t[i] != sc.tokens;
    if (__any_sync(0xffffffffu, bad)) {
        for (int c = i; c < sc.ncounts; c += 32) sc.counts[c] = 0;
        if (i == 0) atomicOr(sc.flags, MOE_FLAG_UNIFORM_SHAPE_DEV);
    }
}
__global__ void fill_i64_kernel(long long* p, long long v) {
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x == 0) *p = v;
}
void launch_fill_i64(long long* p, long long v, cudaStream_t st) {
    launch_pdl(fill_i64_kernel, dim3(1), dim3(32), 0, st, p, v);
}
void launch_ep_shape_check(const long long* all_t, int ep, const ShapeCheck& sc, cudaStream_t st) {
    launch_pdl(ep_shape_check_kernel, dim3(1), dim3(32), 0, st, all_t, ep, sc);
}

// dst += src (the accumulate mode of moe_backward_ex for the non-weight grads)
template <class T>
__global__ void add_into_kernel(T* __restrict__ dst, const T* __restrict__ src, int64_t n) {
    pdl_wait();
    pdl_trigger();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = from_f<T>(to_f(dst[i]) + to_f(src[i]));
}

void launch_add_into(void* dst, const void* src, int64_t n, bool bf16, cudaStream_t st) {
    if (n <= 0) return;
    const unsigned g = (unsigned)std::min<int64_t>(4 * kNumSMs, ceil_div(n, (int64_t)256));
    if (bf16)
        launch_pdl(add_into_kernel<__nv_bfloat16>, dim3(g), dim3(256), 0, st, static_cast<__nv_bfloat16*>(dst),
                   static_cast<const __nv_bfloat16*>(src), n);
    else
        launch_pdl(add_into_kernel<float>, dim3(g), dim3(256), 0, st, static_cast<float*>(dst),
                   static_cast<const float*>(src), n);
}

}  // namespace moe
