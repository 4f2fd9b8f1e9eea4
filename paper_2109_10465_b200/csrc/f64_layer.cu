// f64_layer.cu — the reference-precision path: the MoE layer in float64 on
// the device, for callers whose tensors are the reference's f64 Tensors
// (the tape adapter of INTEGRATION.md §1; gradient checks at h = 1e-5).
//
// Every forward reduction runs in the reference's order with separately
// rounded products and sums (__dmul_rn / __dadd_rn: the reference's x86-64
// build has no FMA contraction), so the gate logits, the expert FFN and the
// combine reproduce routing.cpp / ops.cpp bit for bit; softmax differs from
// glibc exp by at most an ulp.  The backward follows the tape's closures
// (ops.cpp / routing.cpp) to ~1e-15 relative.  Simple
// one-thread-per-output kernels: this path is for parity, the bf16 tcgen05
// path (gemm_tc.cu) is for throughput.
#include "common.cuh"
#include "kernels.h"

namespace moe {
namespace f64 {

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }

__device__ __forceinline__ bool finite_d(double v) { return isfinite(v); }

// Rng::uniform(lo, hi) = lo + (hi - lo) * ((mt() >> 11) * 2^-53), rng.cpp:36-43
__global__ void noise_kernel(uint64_t* buf, int64_t n, double lo, double span) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double u = (double)(buf[i] >> 11) * 0x1.0p-53;
    reinterpret_cast<double*>(buf)[i] = add(lo, mul(span, u));
}

// logits L = (x * noise) Wg; matmul_acc order (ops.cpp:16-29), mul() of the
// jitter first (ops.cpp:213-220)
__global__ void logits_kernel(const double* __restrict__ x, const double* __restrict__ noise,
                              const double* __restrict__ gw, double* __restrict__ L, int64_t T, int d, int E) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= T * E) return;
    const int64_t t = i / E;
    const int e = (int)(i % E);
    double acc = 0.0;
    for (int j = 0; j < d; ++j) {
        const double g = noise ? mul(x[t * d + j], noise[t * d + j]) : x[t * d + j];
        acc = add(acc, mul(g, gw[(int64_t)j * E + e]));
    }
    L[i] = acc;
}

// softmax_row (ops.cpp:77-90), top-1 / top-2 with the reference's tie rules
// (routing.cpp:77-92), pick_per_row, the balance-loss row check
// (routing.cpp:356-363) and the finiteness check of tensor.cpp:23-29.
__global__ void softmax_topk_kernel(const double* __restrict__ L, double* __restrict__ P, int64_t T, int E, int K,
                                    int32_t* __restrict__ choice, double* __restrict__ gp,
                                    uint32_t* __restrict__ flags) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    const double* l = L + t * E;
    double* p = P + t * E;
    uint32_t fl = 0;
    double mx = l[0];
    for (int e = 1; e < E; ++e) mx = fmax(mx, l[e]);
    double sum = 0.0;
    for (int e = 0; e < E; ++e) {
        p[e] = exp(l[e] - mx);
        sum = add(sum, p[e]);
    }
    double s = 0.0;
    for (int e = 0; e < E; ++e) {
        p[e] = p[e] / sum;
        if (!finite_d(p[e]) || !finite_d(l[e])) fl |= MOE_FLAG_NONFINITE_DEV;
        s = add(s, p[e]);
    }
    if (fabs(s - 1.0) > 1e-9) fl |= MOE_FLAG_PROB_ROWS_DEV;
    int best = 0;
    for (int e = 1; e < E; ++e)
        if (p[e] > p[best]) best = e;
    choice[t * K] = best;
    gp[t * K] = p[best];
    if (K == 2) {
        int second = best == 0 ? 1 : 0;
        for (int e = 0; e < E; ++e) {
            if (e == best) continue;
            if (p[e] > p[second]) second = e;
        }
        choice[t * K + 1] = second;
        gp[t * K + 1] = p[second];
    }
    if (fl) atomicOr(flags, fl);
}

// balance_loss (routing.cpp:348-374): f_e = (count of first choices) * alpha E / T,
// aux = dot_constant(mean_cols(P), f) (ops.cpp:513-560); fcoef[e] = f_e / T is
// the per-element gradient of mean_cols (ops.cpp:528-537).  One CTA.
__global__ void balance_kernel(const double* __restrict__ P, const int32_t* __restrict__ choice, int64_t T, int E,
                               int K, double alpha, double* __restrict__ aux, double* __restrict__ fval) {
    extern __shared__ double sh[];  // [E] means
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        double m = 0.0, cnt = 0.0;
        for (int64_t t = 0; t < T; ++t) {
            m = add(m, P[t * E + e]);
            if (choice[t * K] == e) cnt = add(cnt, 1.0);
        }
        sh[e] = m / (double)T;
        const double coeff = mul(alpha, (double)E) / (double)T;
        fval[e] = mul(cnt, coeff);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int e = 0; e < E; ++e) s = add(s, mul(sh[e], fval[e]));
        *aux = s;
    }
}

// combine weights (routing.cpp:408-417): top-1 scale(p, E); top-2 p_k / (p0 + p1)
__global__ void weights_kernel(const double* __restrict__ gp, int64_t T, int E, int K, double* __restrict__ w) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    if (K == 1) {
        w[t] = mul(gp[t], (double)E);
    } else {
        const double tot = add(gp[2 * t], gp[2 * t + 1]);
        w[2 * t] = gp[2 * t] / tot;
        w[2 * t + 1] = gp[2 * t + 1] / tot;
    }
}

// dispatch (routing.cpp:208-243) into the compact [E, cap_pad, d] layout
__global__ void dispatch_kernel(const double* __restrict__ x, int64_t d, int E, int K, int cap_pad,
                                const int32_t* __restrict__ row_src, const int32_t* __restrict__ kept,
                                double* __restrict__ X) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)E * cap_pad * d) return;
    const int64_t r = i / d;
    const int e = (int)(r / cap_pad), p = (int)(r % cap_pad);
    if (p >= kept[e]) return;
    X[i] = x[(int64_t)(row_src[r] / K) * d + (i % d)];
}

// Expert rows: C[r, n] = epi(sum_k A[r, k] W_e(k, n)), r in segment e below kept[e].
// W_e(k, n) = W[e K N + k N + n] (n-major) or W[e N K + n K + k] (k-major).
// epi: 0 none, 1 + bias, 2 + bias then relu (add_bias + relu, ops.cpp:62-75),
// 3 relu mask: C = acc where M[r, n] > 0 else 0 (relu bwd, ops.cpp:307-315).
__global__ void seg_gemm_kernel(const double* __restrict__ A, const double* __restrict__ W, double* __restrict__ C,
                                const double* __restrict__ bias, const double* __restrict__ M,
                                const int32_t* __restrict__ kept, int E, int cap_pad, int64_t K, int64_t N,
                                bool nmajor, int epi) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)E * cap_pad * N) return;
    const int64_t r = i / N, n = i % N;
    const int e = (int)(r / cap_pad);
    if ((int)(r % cap_pad) >= kept[e]) return;
    const double* a = A + r * K;
    const double* w = W + (int64_t)e * K * N;
    double acc = 0.0;
    if (nmajor)
        for (int64_t k = 0; k < K; ++k) acc = add(acc, mul(a[k], w[k * N + n]));
    else
        for (int64_t k = 0; k < K; ++k) acc = add(acc, mul(a[k], w[n * K + k]));
    if (epi == 1 || epi == 2) acc = add(acc, bias[(int64_t)e * N + n]);
    if (epi == 2) acc = acc > 0.0 ? acc : 0.0;
    if (epi == 3) acc = M[i] > 0.0 ? acc : 0.0;
    C[i] = acc;
}

// dW_e[m][n] = sum over the segment's rows of A[r][m] B[r][n] (matmul_at_acc,
// ops.cpp:47-60); db_e[n] = sum over rows of B[r][n] when A == nullptr
// (add_bias bwd, ops.cpp:199-209).  Written, or accumulated with `acc`.
__global__ void seg_wgrad_kernel(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C,
                                 const int32_t* __restrict__ kept, int E, int cap_pad, int64_t Mdim, int64_t N,
                                 bool accumulate) {
    const int64_t Mx = A ? Mdim : 1;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)E * Mx * N) return;
    const int e = (int)(i / (Mx * N));
    const int64_t m = (i / N) % Mx, n = i % N;
    const int64_t r0 = (int64_t)e * cap_pad;
    double acc = 0.0;
    for (int r = 0; r < kept[e]; ++r) {
        const double b = B[(r0 + r) * N + n];
        acc = add(acc, A ? mul(A[(r0 + r) * Mdim + m], b) : b);
    }
    C[i] = accumulate ? add(C[i], acc) : acc;
}

// combine (routing.cpp:279-298): y[t] = sum_{k kept} w_k O[row] (from 0, k order)
// or the residual when no route is kept
__global__ void combine_kernel(const double* __restrict__ O, const double* __restrict__ res, int64_t T, int64_t d,
                               int K, int cap_pad, const int32_t* __restrict__ choice,
                               const int32_t* __restrict__ pos, const double* __restrict__ w,
                               double* __restrict__ y, uint32_t* __restrict__ flags) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= T * d) return;
    const int64_t t = i / d, j = i % d;
    double acc = 0.0;
    bool any = false;
    for (int k = 0; k < K; ++k) {
        const int32_t p = pos[t * K + k];
        if (p < 0) continue;
        any = true;
        const int64_t row = (int64_t)choice[t * K + k] * cap_pad + p;
        acc = add(acc, mul(w[t * K + k], O[row * d + j]));
    }
    const double v = any ? acc : res[i];
    y[i] = v;
    if (!finite_d(v)) atomicOr(flags, MOE_FLAG_NONFINITE_DEV);
}

// combine backward (routing.cpp:311-344): dO rows = w dy[t]; dw_k = <dy[t], O[row]>
__global__ void combine_bwd_kernel(const double* __restrict__ dy, const double* __restrict__ O, int64_t T, int64_t d,
                                   int K, int cap_pad, const int32_t* __restrict__ choice,
                                   const int32_t* __restrict__ pos, const double* __restrict__ w,
                                   double* __restrict__ dO, double* __restrict__ dw) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    for (int k = 0; k < K; ++k) {
        const int32_t p = pos[t * K + k];
        double dot = 0.0;
        if (p >= 0) {
            const int64_t row = (int64_t)choice[t * K + k] * cap_pad + p;
            const double wk = w[t * K + k];
            for (int64_t j = 0; j < d; ++j) {
                dO[row * d + j] = mul(wk, dy[t * d + j]);
                dot = add(dot, mul(dy[t * d + j], O[row * d + j]));
            }
        }
        dw[t * K + k] = dot;
    }
}

// weights / pick / balance / softmax backward -> dL (ops.cpp:250-283, 579-585,
// 552-558, 528-537, 329-343)
__global__ void router_bwd_kernel(const double* __restrict__ P, const double* __restrict__ gp,
                                  const double* __restrict__ dw, const int32_t* __restrict__ choice,
                                  const double* __restrict__ fval, double daux, int64_t T, int E, int K,
                                  double* __restrict__ dL) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    double dp[2] = {0.0, 0.0};
    if (K == 1) {
        dp[0] = mul((double)E, dw[t]);
    } else {
        const double p0 = gp[2 * t], p1 = gp[2 * t + 1];
        const double tot = add(p0, p1);
        double dtot = 0.0;
        for (int k = 0; k < 2; ++k) {
            const double pk = k ? p1 : p0;
            dp[k] = dw[2 * t + k] / tot;
            dtot = dtot - mul(dw[2 * t + k], pk) / mul(tot, tot);
        }
        dp[0] = add(dp[0], dtot);
        dp[1] = add(dp[1], dtot);
    }
    const double inv_t = 1.0 / (double)T;
    const double* p = P + t * E;
    double dot = 0.0;
    for (int e = 0; e < E; ++e) {
        double g = mul(mul(daux, fval[e]), inv_t);
        for (int k = 0; k < K; ++k)
            if (choice[t * K + k] == e) g = add(g, dp[k]);
        dL[t * E + e] = g;  // dP for now
        dot = add(dot, mul(g, p[e]));
    }
    for (int e = 0; e < E; ++e) dL[t * E + e] = mul(p[e], dL[t * E + e] - dot);
}

// gate backward: dWg[j][e] = sum_t g[t][j] dL[t][e] (matmul_at_acc) with
// g = x * noise; one thread per (j, e)
__global__ void gate_dw_kernel(const double* __restrict__ x, const double* __restrict__ noise,
                               const double* __restrict__ dL, double* __restrict__ dW, int64_t T, int d, int E,
                               bool accumulate) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)d * E) return;
    const int j = (int)(i / E), e = (int)(i % E);
    double acc = 0.0;
    for (int64_t t = 0; t < T; ++t) {
        const double g = noise ? mul(x[t * d + j], noise[t * d + j]) : x[t * d + j];
        acc = add(acc, mul(g, dL[t * E + e]));
    }
    dW[i] = accumulate ? add(dW[i], acc) : acc;
}

// dx[t][j] = (sum_e dL[t][e] Wg[j][e]) * noise[t][j]  (matmul_bt_acc + mul bwd)
//          + sum_{k kept} dX[row_k][j]               (dispatch bwd, routing.cpp:245-253)
//          + dy[t][j] if no route kept and the residual is x; else dres = dy there
__global__ void dx_kernel(const double* __restrict__ dL, const double* __restrict__ gw,
                          const double* __restrict__ noise, const double* __restrict__ dX,
                          const double* __restrict__ dy, int64_t T, int d, int E, int K, int cap_pad,
                          const int32_t* __restrict__ choice, const int32_t* __restrict__ pos,
                          bool residual_is_x, double* __restrict__ dx, double* __restrict__ dres,
                          bool accumulate) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= T * d) return;
    const int64_t t = i / d;
    const int j = (int)(i % d);
    double g = 0.0;
    for (int e = 0; e < E; ++e) g = add(g, mul(dL[t * E + e], gw[(int64_t)j * E + e]));
    if (noise) g = mul(g, noise[i]);
    bool any = false;
    for (int k = 0; k < K; ++k) {
        const int32_t p = pos[t * K + k];
        if (p < 0) continue;
        any = true;
        g = add(g, dX[((int64_t)choice[t * K + k] * cap_pad + p) * d + j]);
    }
    if (!any && residual_is_x) g = add(g, dy[i]);
    dx[i] = accumulate ? add(dx[i], g) : g;
    if (dres) {
        const double r = any ? 0.0 : dy[i];
        dres[i] = accumulate ? add(dres[i], r) : r;
    }
}

__global__ void acc_copy_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t n,
                                bool accumulate) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = accumulate ? add(dst[i], src[i]) : src[i];
}

inline unsigned blocks(int64_t n) { return (unsigned)ceil_div(n, (int64_t)256); }

}  // namespace f64

void launch_f64_noise(uint64_t* buf, int64_t n, double lo, double hi, cudaStream_t st) {
    if (n <= 0) return;
    f64::noise_kernel<<<f64::blocks(n), 256, 0, st>>>(buf, n, lo, hi - lo);
    MOE_LAUNCH_CHECK();
}
void launch_f64_gate(const double* x, const double* noise, const double* gw, double* L, double* P, int64_t T,
                     int d, int E, int K, int32_t* choice, double* gp, uint32_t* flags, cudaStream_t st) {
    f64::logits_kernel<<<f64::blocks(T * E), 256, 0, st>>>(x, noise, gw, L, T, d, E);
    MOE_LAUNCH_CHECK();
    f64::softmax_topk_kernel<<<f64::blocks(T), 256, 0, st>>>(L, P, T, E, K, choice, gp, flags);
    MOE_LAUNCH_CHECK();
}
void launch_f64_balance(const double* P, const int32_t* choice, int64_t T, int E, int K, double alpha,
                        double* aux, double* fval, cudaStream_t st) {
    f64::balance_kernel<<<1, 256, sizeof(double) * E, st>>>(P, choice, T, E, K, alpha, aux, fval);
    MOE_LAUNCH_CHECK();
}
void launch_f64_weights(const double* gp, int64_t T, int E, int K, double* w, cudaStream_t st) {
    f64::weights_kernel<<<f64::blocks(T), 256, 0, st>>>(gp, T, E, K, w);
    MOE_LAUNCH_CHECK();
}
void launch_f64_dispatch(const double* x, int64_t d, int E, int K, int cap_pad, const int32_t* row_src,
                         const int32_t* kept, double* X, cudaStream_t st) {
    f64::dispatch_kernel<<<f64::blocks((int64_t)E * cap_pad * d), 256, 0, st>>>(x, d, E, K, cap_pad, row_src,
                                                                               kept, X);
    MOE_LAUNCH_CHECK();
}
void launch_f64_seg_gemm(const double* A, const double* W, double* C, const double* bias, const double* M,
                         const int32_t* kept, int E, int cap_pad, int64_t K, int64_t N, bool nmajor, int epi,
                         cudaStream_t st) {
    f64::seg_gemm_kernel<<<f64::blocks((int64_t)E * cap_pad * N), 256, 0, st>>>(A, W, C, bias, M, kept, E,
                                                                                cap_pad, K, N, nmajor, epi);
    MOE_LAUNCH_CHECK();
}
void launch_f64_seg_wgrad(const double* A, const double* B, double* C, const int32_t* kept, int E, int cap_pad,
                          int64_t M, int64_t N, bool accumulate, cudaStream_t st) {
    const int64_t Mx = A ? M : 1;
    f64::seg_wgrad_kernel<<<f64::blocks((int64_t)E * Mx * N), 256, 0, st>>>(A, B, C, kept, E, cap_pad, M, N,
                                                                            accumulate);
    MOE_LAUNCH_CHECK();
}
void launch_f64_combine(const double* O, const double* res, int64_t T, int64_t d, int K, int cap_pad,
                        const int32_t* choice, const int32_t* pos, const double* w, double* y,
                        uint32_t* flags, cudaStream_t st) {
    f64::combine_kernel<<<f64::blocks(T * d), 256, 0, st>>>(O, res, T, d, K, cap_pad, choice, pos, w, y, flags);
    MOE_LAUNCH_CHECK();
}
void launch_f64_combine_bwd(const double* dy, const double* O, int64_t T, int64_t d, int K, int cap_pad,
                            const int32_t* choice, const int32_t* pos, const double* w, double* dO, double* dw,
                            cudaStream_t st) {
    f64::combine_bwd_kernel<<<f64::blocks(T), 256, 0, st>>>(dy, O, T, d, K, cap_pad, choice, pos, w, dO, dw);
    MOE_LAUNCH_CHECK();
}
void launch_f64_router_bwd(const double* P, const double* gp, const double* dw, const int32_t* choice,
                           const double* fval, double daux, int64_t T, int E, int K, double* dL,
                           cudaStream_t st) {
    f64::router_bwd_kernel<<<f64::blocks(T), 256, 0, st>>>(P, gp, dw, choice, fval, daux, T, E, K, dL);
    MOE_LAUNCH_CHECK();
}
void launch_f64_gate_dw(const double* x, const double* noise, const double* dL, double* dW, int64_t T, int d,
                        int E, bool accumulate, cudaStream_t st) {
    f64::gate_dw_kernel<<<f64::blocks((int64_t)d * E), 256, 0, st>>>(x, noise, dL, dW, T, d, E, accumulate);
    MOE_LAUNCH_CHECK();
}
void launch_f64_dx(const double* dL, const double* gw, const double* noise, const double* dX, const double* dy,
                   int64_t T, int d, int E, int K, int cap_pad, const int32_t* choice, const int32_t* pos,
                   bool residual_is_x, double* dx, double* dres, bool accumulate, cudaStream_t st) {
    f64::dx_kernel<<<f64::blocks(T * d), 256, 0, st>>>(dL, gw, noise, dX, dy, T, d, E, K, cap_pad, choice, pos,
                                                       residual_is_x, dx, dres, accumulate);
    MOE_LAUNCH_CHECK();
}
void launch_f64_acc_copy(const double* src, double* dst, int64_t n, bool accumulate, cudaStream_t st) {
    if (n <= 0) return;
    f64::acc_copy_kernel<<<f64::blocks(n), 256, 0, st>>>(src, dst, n, accumulate);
    MOE_LAUNCH_CHECK();
}

}  // namespace moe
