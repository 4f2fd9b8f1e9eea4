// gemm_simt.cu — fp32-accumulating SIMT GEMMs.
//
// Used for (a) the fp32 parity path of the expert FFN (the reference runs the
// expert FFN in f64, routing.cpp:397-406 / ops.cpp:16-60; 1e-5 relative needs
// fp32 FFMA, not bf16 tensor cores) and (b) the small gate GEMMs
// (logits = (x*noise) Wg, dx_gate = dL Wg^T, dWg = g^T dL; ops.cpp:125-144).
// The bf16 expert GEMMs run on tcgen05 (gemm_tc.cu).
//
// One 64x64 output tile per CTA, K staged through shared memory 16 at a time,
// 256 threads with 4x4 register micro-tiles.  Reductions are in a fixed order
// (deterministic).
#include "common.cuh"
#include "kernels.h"

namespace moe {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

struct Acc {
    float v[4][4];
};

__device__ __forceinline__ void tile_fma(const float (*As)[BM + 4], const float (*Bs)[BN + 4],
                                         Acc& acc, int tm, int tn) {
#pragma unroll
    for (int k = 0; k < BK; ++k) {
        const float4 a = *reinterpret_cast<const float4*>(&As[k][tm]);
        const float4 b = *reinterpret_cast<const float4*>(&Bs[k][tn]);
        const float av[4] = {a.x, a.y, a.z, a.w};
        const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc.v[i][j] = fmaf(av[i], bv[j], acc.v[i][j]);
    }
}

// ---------------------------------------------------------------------------
// dense strided GEMM (gate GEMMs)
// ---------------------------------------------------------------------------
template <class TA>
__global__ void __launch_bounds__(NT)
gemm_dense_kernel(const TA* __restrict__ A, int64_t lda_m, int64_t lda_k,
                  const float* __restrict__ S, const float* __restrict__ B, int64_t ldb_k,
                  int64_t ldb_n, float* __restrict__ C, int64_t M, int64_t N, int64_t K,
                  int64_t k_per_split) {
    pdl_wait();
    pdl_trigger();
    __shared__ __align__(16) float As[BK][BM + 4];
    __shared__ __align__(16) float Bs[BK][BN + 4];
    const int tid = threadIdx.x;
    const int tm = (tid / 16) * 4, tn = (tid % 16) * 4;
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
    const int64_t kb = (int64_t)blockIdx.z * k_per_split;
    const int64_t ke = min(K, kb + k_per_split);
    const bool a_kc = lda_k == 1;  // K contiguous in A
    const bool b_nc = ldb_n == 1;  // N contiguous in B
    Acc acc = {};
    for (int64_t k0 = kb; k0 < ke; k0 += BK) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int idx = tid + i * NT;
            int mm, kk;
            if (a_kc) { mm = idx / BK; kk = idx % BK; } else { mm = idx % BM; kk = idx / BM; }
            const int64_t gm = m0 + mm, gk = k0 + kk;
            float v = 0.f;
            if (gm < M && gk < ke) {
                const int64_t off = gm * lda_m + gk * lda_k;
                v = to_f(A[off]);
                if (S) v *= S[off];
            }
            As[kk][mm] = v;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int idx = tid + i * NT;
            int nn, kk;
            if (b_nc) { nn = idx % BN; kk = idx / BN; } else { nn = idx / BK; kk = idx % BK; }
            const int64_t gn = n0 + nn, gk = k0 + kk;
            Bs[kk][nn] = (gn < N && gk < ke) ? B[gk * ldb_k + gn * ldb_n] : 0.f;
        }
        __syncthreads();
        tile_fma(As, Bs, acc, tm, tn);
        __syncthreads();
    }
    float* Cz = C + (int64_t)blockIdx.z * M * N;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t gm = m0 + tm + i, gn = n0 + tn + j;
            if (gm < M && gn < N) Cz[gm * N + gn] = acc.v[i][j];
        }
}

template <class TA>
void launch_gemm_dense(const TA* A, int64_t lda_m, int64_t lda_k, const float* S, const float* B,
                       int64_t ldb_k, int64_t ldb_n, float* C, int64_t M, int64_t N, int64_t K,
                       int split_k, cudaStream_t st) {
    if (M == 0 || N == 0) return;
    const int64_t kps = round_up(ceil_div(K, split_k), BK);
    dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, BM), (unsigned)split_k);
    launch_pdl(gemm_dense_kernel<TA>, dim3(grid), dim3(NT), 0, st, A, lda_m, lda_k, S, B, ldb_k, ldb_n, C, M, N, K,
                                               kps);
}

__global__ void splitk_reduce_kernel(const float* __restrict__ part, int split_k, int64_t MN,
                                     float* __restrict__ out) {
    pdl_wait();
    pdl_trigger();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= MN) return;
    float acc = 0.f;
    for (int s = 0; s < split_k; ++s) acc += part[(int64_t)s * MN + i];
    out[i] = acc;
}

void launch_splitk_reduce(const float* part, int split_k, int64_t MN, float* out,
                          cudaStream_t st) {
    launch_pdl(splitk_reduce_kernel, dim3((unsigned)ceil_div(MN, 256)), dim3(256), 0, st, part, split_k, MN, out);
}

template void launch_gemm_dense<float>(const float*, int64_t, int64_t, const float*,
                                       const float*, int64_t, int64_t, float*, int64_t, int64_t,
                                       int64_t, int, cudaStream_t);
template void launch_gemm_dense<__nv_bfloat16>(const __nv_bfloat16*, int64_t, int64_t,
                                               const float*, const float*, int64_t, int64_t,
                                               float*, int64_t, int64_t, int64_t, int,
                                               cudaStream_t);

// ---------------------------------------------------------------------------
// expert GEMM over buffer rows (fwd1, fwd2, dgrad2, dgrad1)
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(NT)
row_gemm_simt_kernel(RowGemmArgs a) {
    pdl_wait();
    pdl_trigger();
    __shared__ __align__(16) float As[BK][BM + 4];
    __shared__ __align__(16) float Bs[BK][BN + 4];
    const int seg = blockIdx.z;             // r * El + le
    const int le = seg % a.El;
    const int count = a.counts[seg];
    const int64_t mt0 = (int64_t)blockIdx.y * BM;  // row offset inside the segment
    if (mt0 >= round_up_dev(count, kRowAlign)) return;
    const int64_t row0 = (int64_t)seg * a.cap_pad + mt0;
    const int64_t n0 = (int64_t)blockIdx.x * BN;
    const int64_t N = a.N, K = a.K;
    const T* A = static_cast<const T*>(a.A);
    const T* W = static_cast<const T*>(a.W) + (int64_t)le * N * K;
    T* C = static_cast<T*>(a.C);
    const int tid = threadIdx.x;
    const int tm = (tid / 16) * 4, tn = (tid % 16) * 4;
    Acc acc = {};
    const bool compute = mt0 < count;
    for (int64_t k0 = 0; compute && k0 < K; k0 += BK) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int idx = tid + i * NT;
            const int mm = idx / BK, kk = idx % BK;
            const int64_t gk = k0 + kk;
            As[kk][mm] = (mt0 + mm < count && gk < K) ? to_f(A[(row0 + mm) * K + gk]) : 0.f;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int idx = tid + i * NT;
            int nn, kk;
            if (a.w_nmajor) { nn = idx % BN; kk = idx / BN; } else { nn = idx / BK; kk = idx % BK; }
            const int64_t gn = n0 + nn, gk = k0 + kk;
            float v = 0.f;
            if (gn < N && gk < K) v = to_f(a.w_nmajor ? W[gk * N + gn] : W[gn * K + gk]);
            Bs[kk][nn] = v;
        }
        __syncthreads();
        tile_fma(As, Bs, acc, tm, tn);
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t m = mt0 + tm + i;
        if (m >= round_up_dev(count, kRowAlign)) continue;
        const bool valid = m < count;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t gn = n0 + tn + j;
            if (gn >= N) continue;
            float v = 0.f;
            if (valid) {
                v = acc.v[i][j];
                if (a.epi == EPI_BIAS || a.epi == EPI_BIAS_RELU) v += a.bias[(int64_t)le * N + gn];
                if (a.epi == EPI_BIAS_RELU) v = v > 0.f ? v : 0.f;
                if (a.epi == EPI_RELU_MASK) {
                    const float h = to_f(static_cast<const T*>(a.mask)[((int64_t)seg * a.cap_pad + m) * N + gn]);
                    if (!(h > 0.f)) v = 0.f;
                }
            }
            C[((int64_t)seg * a.cap_pad + m) * N + gn] = from_f<T>(v);
        }
    }
}

template <class T>
void launch_row_gemm_simt(const RowGemmArgs& a, cudaStream_t st) {
    dim3 grid((unsigned)ceil_div(a.N, BN), (unsigned)ceil_div(a.cap_pad, BM), (unsigned)(a.ep * a.El));
    launch_pdl(row_gemm_simt_kernel<T>, dim3(grid), dim3(NT), 0, st, a);
}

// ---------------------------------------------------------------------------
// expert weight gradient: C_g = sum over the group's rows of A[row,:]^T B[row,:]
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(NT)
wgrad_gemm_simt_kernel(WgradGemmArgs a) {
    pdl_wait();
    pdl_trigger();
    __shared__ __align__(16) float As[BK][BM + 4];
    __shared__ __align__(16) float Bs[BK][BN + 4];
    const int g = blockIdx.z;
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
    const int64_t M = a.M, N = a.N;
    const T* A = static_cast<const T*>(a.A);
    const T* B = static_cast<const T*>(a.B);
    const int tid = threadIdx.x;
    const int tm = (tid / 16) * 4, tn = (tid % 16) * 4;
    Acc acc = {};
    for (int r = 0; r < a.ep; ++r) {
        const int seg = r * a.El + g;
        const int count = a.counts[seg];
        const int64_t rbase = (int64_t)seg * a.cap_pad;
        for (int k0 = 0; k0 < count; k0 += BK) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int idx = tid + i * NT;
                const int mm = idx % BM, kk = idx / BM;
                const int64_t gm = m0 + mm;
                As[kk][mm] = (gm < M && k0 + kk < count) ? to_f(A[(rbase + k0 + kk) * M + gm]) : 0.f;
                const int64_t gn = n0 + mm;  // BN == BM
                Bs[kk][mm] = (gn < N && k0 + kk < count) ? to_f(B[(rbase + k0 + kk) * N + gn]) : 0.f;
            }
            __syncthreads();
            tile_fma(As, Bs, acc, tm, tn);
            __syncthreads();
        }
    }
    const bool add = a.c_mode & 1;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t gm = m0 + tm + i, gn = n0 + tn + j;
            if (gm >= M || gn >= N) continue;
            const int64_t o = (int64_t)g * M * N + gm * N + gn;
            if (a.c_mode & 2) {  // fp32 output
                float* C = static_cast<float*>(a.C);
                C[o] = add ? C[o] + acc.v[i][j] : acc.v[i][j];
            } else {
                T* C = static_cast<T*>(a.C);
                C[o] = from_f<T>(add ? to_f(C[o]) + acc.v[i][j] : acc.v[i][j]);
            }
        }
}

template <class T>
void launch_wgrad_gemm_simt(const WgradGemmArgs& a, cudaStream_t st) {
    dim3 grid((unsigned)ceil_div(a.N, BN), (unsigned)ceil_div(a.M, BM), (unsigned)a.El);
    launch_pdl(wgrad_gemm_simt_kernel<T>, dim3(grid), dim3(NT), 0, st, a);
}

template void launch_row_gemm_simt<float>(const RowGemmArgs&, cudaStream_t);
template void launch_row_gemm_simt<__nv_bfloat16>(const RowGemmArgs&, cudaStream_t);
template void launch_wgrad_gemm_simt<float>(const WgradGemmArgs&, cudaStream_t);
template void launch_wgrad_gemm_simt<__nv_bfloat16>(const WgradGemmArgs&, cudaStream_t);

}  // namespace moe
