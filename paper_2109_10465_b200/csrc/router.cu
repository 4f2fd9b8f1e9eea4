// router.cu — gate softmax/top-k, capacity-slot assignment scan and the
// balance-loss reduction (forward and backward) for the B200 MoE layer.
//
// Reference semantics (paths relative to /root/reference/proj/core):
//   gate_forward       src/routing.cpp:51-101
//   scan_assign & co.  src/routing.cpp:113-206
//   balance_loss       src/routing.cpp:348-374 (mean_cols ops.cpp:513-539,
//                      dot_constant ops.cpp:541-560)
//   softmax backward   src/ops.cpp:329-343; pick_per_row bwd ops.cpp:579-585;
//                      scale/add/div_elem bwd ops.cpp:250-281
#include "common.cuh"
#include "kernels.h"

namespace moe {

// ---------------------------------------------------------------------------
// softmax + top-k over one row of logits per warp.
//   P = exp(L - max) / sum (ops.cpp:77-90)
//   c0 = argmax_e P (strict >, lowest index wins), c1 = argmax over e != c0
//   with the candidate initialised to (c0 == 0 ? 1 : 0) (routing.cpp:77-92).
// Also: per-CTA partial column sums of P and first-choice histograms for the
// balance loss (fixed-order reduction in balance_finalize), and latched
// flags for non-finite values / rows not summing to one.
// ---------------------------------------------------------------------------
constexpr int kSoftmaxWarps = 8;
constexpr int kRowsPerPart = 2 * kSoftmaxWarps;  // token rows per CTA (2 per warp)

// NL = logits per lane (E <= 32 NL), NS = split-K partial arrays: both
// compile-time so every row's loads are issued together.
template <int NL, int NS>
__global__ void __launch_bounds__(kSoftmaxWarps * 32)
softmax_topk_kernel(const float* __restrict__ logits, int64_t T, int E, int K,
                    float* __restrict__ probs, int32_t* __restrict__ choice,
                    float* __restrict__ gate_prob, float* __restrict__ colsum_part,
                    int32_t* __restrict__ count_part, uint32_t* __restrict__ flags) {
    pdl_wait();
    pdl_trigger();
    const int64_t TE = T * E;
    extern __shared__ float sm[];
    float* s_col = sm;                                   // [warps][E]
    int32_t* s_cnt = reinterpret_cast<int32_t*>(sm + kSoftmaxWarps * E);  // [E]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < kSoftmaxWarps * E; i += blockDim.x) s_col[i] = 0.f;
    for (int i = threadIdx.x; i < E; i += blockDim.x) s_cnt[i] = 0;
    __syncthreads();
    uint32_t flag = 0;
    const int64_t rows_per_cta = kRowsPerPart;
    const int64_t t0 = (int64_t)blockIdx.x * rows_per_cta;
    for (int64_t t = t0 + warp; t < min(T, t0 + rows_per_cta); t += kSoftmaxWarps) {
        const float* Lp = logits + t * E;
        float part[NL][NS];  // split-K partials, loaded together, summed in fixed order
#pragma unroll
        for (int q = 0; q < NL; ++q)
#pragma unroll
            for (int s2 = 0; s2 < NS; ++s2)
                part[q][s2] = lane + 32 * q < E ? __ldg(Lp + s2 * TE + lane + 32 * q) : 0.f;
        float L[NL];
#pragma unroll
        for (int q = 0; q < NL; ++q) {
            float v = part[q][0];
#pragma unroll
            for (int s2 = 1; s2 < NS; ++s2) v += part[q][s2];
            L[q] = v;
        }
        float mx = -INFINITY;
#pragma unroll
        for (int q = 0; q < NL; ++q)
            if (lane + 32 * q < E) mx = fmaxf(mx, L[q]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float s = 0.f;
#pragma unroll
        for (int q = 0; q < NL; ++q)
            if (lane + 32 * q < E) s += expf(L[q] - mx);
        s = warp_sum(s);
        // best / second best over P with the reference's tie rules
        float b0 = -1.f, b1 = -1.f;
        int i0 = 0x7fffffff, i1 = 0x7fffffff;
        float psum = 0.f;
#pragma unroll
        for (int q = 0; q < NL; ++q) {
            const int e = lane + 32 * q;
            if (e >= E) continue;
            const float p = expf(L[q] - mx) / s;
            probs[t * E + e] = p;
            s_col[warp * E + e] += p;
            psum += p;
            if (!finite_f(p) || !finite_f(L[q])) flag |= MOE_FLAG_NONFINITE_DEV;
            // keep the two best (value desc, index asc) seen by this lane
            if (p > b0 || (p == b0 && e < i0)) {
                b1 = b0; i1 = i0; b0 = p; i0 = e;
            } else if (p > b1 || (p == b1 && e < i1)) {
                b1 = p; i1 = e;
            }
        }
        psum = warp_sum(psum);
        // warp merge of (b0,i0,b1,i1)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float ob0 = __shfl_xor_sync(0xffffffffu, b0, o);
            const int oi0 = __shfl_xor_sync(0xffffffffu, i0, o);
            const float ob1 = __shfl_xor_sync(0xffffffffu, b1, o);
            const int oi1 = __shfl_xor_sync(0xffffffffu, i1, o);
            // merge two sorted pairs
            float c[4] = {b0, b1, ob0, ob1};
            int ci[4] = {i0, i1, oi0, oi1};
            float nb0 = -1.f, nb1 = -1.f;
            int ni0 = 0x7fffffff, ni1 = 0x7fffffff;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float p = c[q];
                const int e = ci[q];
                if (e == ni0) continue;
                if (p > nb0 || (p == nb0 && e < ni0)) {
                    nb1 = nb0; ni1 = ni0; nb0 = p; ni0 = e;
                } else if (e != ni0 && (p > nb1 || (p == nb1 && e < ni1))) {
                    nb1 = p; ni1 = e;
                }
            }
            b0 = nb0; i0 = ni0; b1 = nb1; i1 = ni1;
        }
        if (i0 < 0 || i0 >= E) {  // NaN row: no comparison succeeded (flagged above)
            i0 = 0;
            b0 = 0.f;
        }
        if (i1 < 0 || i1 >= E || i1 == i0) {
            i1 = i0 == 0 ? 1 % E : 0;
            b1 = 0.f;
        }
        if (lane == 0) {
            choice[t * K] = i0;
            gate_prob[t * K] = b0;
            if (K == 2) {
                choice[t * K + 1] = i1;
                gate_prob[t * K + 1] = b1;
            }
            atomicAdd(&s_cnt[i0], 1);
            if (fabsf(psum - 1.0f) > kProbRowTol) flag |= MOE_FLAG_PROB_ROWS_DEV;
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        float acc = 0.f;
        for (int w = 0; w < kSoftmaxWarps; ++w) acc += s_col[w * E + e];
        colsum_part[(int64_t)blockIdx.x * E + e] = acc;
        count_part[(int64_t)blockIdx.x * E + e] = s_cnt[e];
    }
    flag = __reduce_or_sync(0xffffffffu, flag);
    if (lane == 0 && flag) atomicOr(flags, flag);
}

// aux = sum_e mean_t(P[:,e]) * f_e,  f_e = alpha * E * count_e / T.
// Also emits fcoef[e] = f_e / T, the per-element gradient dP += daux * f_e/T.
// One CTA per expert reduces that expert's per-part partials (fixed order:
// strided per thread, then a shared-memory tree); the last CTA to finish sums
// the E terms in expert order.  Deterministic, no float atomics.
__global__ void __launch_bounds__(256)
balance_finalize_kernel(const float* __restrict__ colsum_part, const int32_t* __restrict__ count_part,
                        int nparts, int64_t T, int E, double alpha, float* __restrict__ aux,
                        float* __restrict__ fcoef, int32_t* __restrict__ counts,
                        double* __restrict__ term, unsigned* __restrict__ done) {
    pdl_wait();
    pdl_trigger();
    __shared__ double s_cs[256];
    __shared__ long long s_cnt[256];
    __shared__ bool last;
    const int e = blockIdx.x;
    double cs = 0.0;
    long long cnt = 0;
    for (int p = threadIdx.x; p < nparts; p += blockDim.x) {
        cs += (double)colsum_part[(int64_t)p * E + e];
        cnt += count_part[(int64_t)p * E + e];
    }
    s_cs[threadIdx.x] = cs;
    s_cnt[threadIdx.x] = cnt;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            s_cs[threadIdx.x] += s_cs[threadIdx.x + o];
            s_cnt[threadIdx.x] += s_cnt[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double f = alpha * (double)E * (double)s_cnt[0] / (double)T;
        if (fcoef) fcoef[e] = (float)(f / (double)T);
        if (counts) counts[e] = (int32_t)s_cnt[0];
        term[e] = (s_cs[0] / (double)T) * f;
        __threadfence();
        last = atomicAdd(done, 1u) == (unsigned)(E - 1);
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        double s = 0.0;
        for (int q = 0; q < E; ++q) s += ((volatile double*)term)[q];
        *aux = (float)s;
        *done = 0u;  // reset for the next call
    }
}

void launch_softmax_topk(const float* logits, int nsplit, int64_t T, int E, int K, float* probs,
                         int32_t* choice, float* gate_prob, float* colsum_part,
                         int32_t* count_part, uint32_t* flags, cudaStream_t st) {
    if (E > 256) throw Status(2, "gate: num_experts > 256 not supported on this path");
    const int nparts = softmax_parts(T);
    const size_t smem = sizeof(float) * kSoftmaxWarps * E + sizeof(int32_t) * E;
    const int nl = E <= 32 ? 1 : E <= 64 ? 2 : E <= 128 ? 4 : 8;
    auto go = [&](auto kernel) {
        launch_pdl(kernel, dim3(nparts), dim3(kSoftmaxWarps * 32), smem, st, logits, T, E, K, probs, choice, gate_prob,
                                                         colsum_part, count_part, flags);
    };
#define MOE_SOFTMAX_NS(NLV)                                                           \
    switch (nsplit) {                                                                 \
        case 1: go(softmax_topk_kernel<NLV, 1>); break;                               \
        case 2: go(softmax_topk_kernel<NLV, 2>); break;                               \
        case 4: go(softmax_topk_kernel<NLV, 4>); break;                               \
        case 8: go(softmax_topk_kernel<NLV, 8>); break;                               \
        default: throw Status(2, "softmax: split-K count must be 1, 2, 4 or 8");      \
    }
    switch (nl) {
        case 1: MOE_SOFTMAX_NS(1) break;
        case 2: MOE_SOFTMAX_NS(2) break;
        case 4: MOE_SOFTMAX_NS(4) break;
        default: MOE_SOFTMAX_NS(8) break;
    }
#undef MOE_SOFTMAX_NS
    MOE_LAUNCH_CHECK();
}

int softmax_parts(int64_t T) { return (int)ceil_div(T, (int64_t)kRowsPerPart); }

void launch_balance_finalize(const float* colsum_part, const int32_t* count_part, int nparts,
                             int64_t T, int E, double alpha, float* aux, float* fcoef,
                             int32_t* counts, double* term, unsigned* done, cudaStream_t st) {
    launch_pdl(balance_finalize_kernel, dim3(E), dim3(256), 0, st, colsum_part, count_part, nparts, T, E, alpha, aux,
                                               fcoef, counts, term, done);
}

// ---------------------------------------------------------------------------
// Slot assignment: an order-dependent scan (routing.cpp:116-145) made
// parallel.  The scan order is a list of positions i -> token ord[i]
// (identity, or the RTS permutation), cut into G contiguous groups (grouped
// mode) that run independently with span = ceil(cap/G) and base g*span.
// Visits are k-major: the k=1 pass starts from the clipped k=0 totals.
//
//   count kernel : per chunk (<=kChunk positions, never straddling a group)
//                  histogram of choices, for each k
//   scan kernel  : per (group, expert), exclusive prefix over the group's
//                  chunks -> chunk bases; group totals -> kept counts and the
//                  compact position base of each group
//   rank kernel  : per chunk, rank of each position among same-expert
//                  positions (warp match_any + per-warp counts) -> slot
//
// Besides the reference slot, each kept route gets a compact position
// pos in [0, kept_e) of its expert (== slot except in grouped mode) and the
// inverse map row_src[e*cap_pad + pos] = t*K + k used by the gather kernels.
// ---------------------------------------------------------------------------
constexpr int kChunk = 1024;

struct ScanGeom {
    int64_t T;
    int G;
    int64_t glen;       // positions per group
    int cpg;            // chunks per group
    int E, K;
    int span;           // per-group capacity
};

__device__ __forceinline__ void chunk_range(const ScanGeom& g, int c, int64_t& b, int64_t& e,
                                            int& grp) {
    grp = c / g.cpg;
    const int j = c % g.cpg;
    b = (int64_t)grp * g.glen + (int64_t)j * kChunk;
    e = min(b + (int64_t)kChunk, (int64_t)(grp + 1) * g.glen);
}

__global__ void __launch_bounds__(kChunk)
assign_count_kernel(ScanGeom g, const int32_t* __restrict__ choice,
                    const uint32_t* __restrict__ ord, int32_t* __restrict__ hist,
                    uint32_t* __restrict__ flags) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ int32_t s_h[];  // [K][E]
    for (int i = threadIdx.x; i < g.K * g.E; i += blockDim.x) s_h[i] = 0;
    __syncthreads();
    int64_t b, e;
    int grp;
    chunk_range(g, blockIdx.x, b, e, grp);
    const int64_t i = b + threadIdx.x;
    if (i < e) {
        const int64_t t = ord ? (int64_t)ord[i] : i;
        for (int k = 0; k < g.K; ++k) {
            const int32_t c = choice[t * g.K + k];
            if (c < 0 || c >= g.E) {
                atomicOr(flags, MOE_FLAG_CHOICE_RANGE_DEV);
                continue;
            }
            atomicAdd(&s_h[k * g.E + c], 1);
        }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < g.K * g.E; q += blockDim.x)
        hist[(int64_t)blockIdx.x * g.K * g.E + q] = s_h[q];
}

// One thread per (group, expert).  base[c][k][e] = slot offset of chunk c's
// first k-route of expert e inside its group (k=1 continues from the clipped
// k=0 total).  gkept[grp][e] = routes kept in the group; gbase[grp][e] =
// compact position of the group's first kept route; kept[e] = sum.
__global__ void assign_scan_kernel(ScanGeom g, const int32_t* __restrict__ hist,
                                   int32_t* __restrict__ base, int32_t* __restrict__ gkept,
                                   int32_t* __restrict__ kept) {
    pdl_wait();
    pdl_trigger();
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= g.E) return;
    int32_t run_compact = 0;
    for (int grp = 0; grp < g.G; ++grp) {
        int32_t run0 = 0;
        for (int j = 0; j < g.cpg; ++j) {
            const int c = grp * g.cpg + j;
            base[((int64_t)c * g.K + 0) * g.E + e] = run0;
            run0 += hist[((int64_t)c * g.K + 0) * g.E + e];
        }
        const int32_t kept0 = min(run0, g.span);
        int32_t kept_g = kept0;
        if (g.K == 2) {
            int32_t run1 = kept0;
            for (int j = 0; j < g.cpg; ++j) {
                const int c = grp * g.cpg + j;
                base[((int64_t)c * g.K + 1) * g.E + e] = run1;
                run1 += hist[((int64_t)c * g.K + 1) * g.E + e];
            }
            kept_g = min(run1, g.span);
        }
        gkept[(int64_t)grp * g.E * 2 + e] = kept_g;        // routes kept in group
        gkept[(int64_t)grp * g.E * 2 + g.E + e] = run_compact;  // compact base
        run_compact += kept_g;
    }
    kept[e] = run_compact;
}

__global__ void __launch_bounds__(kChunk)
assign_rank_kernel(ScanGeom g, const int32_t* __restrict__ choice,
                   const uint32_t* __restrict__ ord, const int32_t* __restrict__ base,
                   const int32_t* __restrict__ gkept, int cap_pad, int32_t* __restrict__ slot,
                   int32_t* __restrict__ pos, int32_t* __restrict__ row_src) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ int32_t s_w[];  // [32 warps][E]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int64_t b, e;
    int grp;
    chunk_range(g, blockIdx.x, b, e, grp);
    const int64_t i = b + threadIdx.x;
    const bool active = i < e;
    const int64_t t = active ? (ord ? (int64_t)ord[i] : i) : 0;
    const unsigned lt_mask = (1u << lane) - 1u;
    for (int k = 0; k < g.K; ++k) {
        for (int q = threadIdx.x; q < 32 * g.E; q += blockDim.x) s_w[q] = 0;
        __syncthreads();
        const int32_t c = active ? choice[t * g.K + k] : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, c);
        const int rank_w = __popc(peers & lt_mask);
        if (active && c >= 0 && c < g.E && rank_w == 0) s_w[warp * g.E + c] = __popc(peers);
        __syncthreads();
        if (active && c >= 0 && c < g.E) {
            int32_t r = rank_w;
            for (int w = 0; w < warp; ++w) r += s_w[w * g.E + c];
            const int32_t local = base[((int64_t)blockIdx.x * g.K + k) * g.E + c] + r;
            const int64_t idx = t * g.K + k;
            if (local < g.span) {
                slot[idx] = grp * g.span + local;
                const int32_t p = gkept[(int64_t)grp * g.E * 2 + g.E + c] + local;
                pos[idx] = p;
                row_src[(int64_t)c * cap_pad + p] = (int32_t)idx;
            } else {
                slot[idx] = -1;
                pos[idx] = -1;
            }
        }
        __syncthreads();
    }
}

void launch_assign(int64_t T, int E, int K, int cap, int mode, int G, const int32_t* choice,
                   const uint32_t* ord, int cap_pad, AssignScratch& s, int32_t* slot, int32_t* pos,
                   int32_t* row_src, int32_t* kept, uint32_t* flags, cudaStream_t st) {
    ScanGeom g;
    g.T = T;
    g.E = E;
    g.K = K;
    if (mode == 1) {  // grouped (routing.cpp:156-178)
        g.G = G;
        g.glen = T / G;
        g.span = (int)((cap + G - 1) / G);
    } else {
        g.G = 1;
        g.glen = T;
        g.span = cap;
        if (mode != 2) ord = nullptr;
    }
    g.cpg = (int)ceil_div(g.glen, kChunk);
    const int nchunks = g.G * g.cpg;
    if (nchunks > s.max_chunks || g.G > s.max_groups)
        throw Status(1, "assign: scratch too small");
    launch_pdl(assign_count_kernel, dim3(nchunks), dim3(kChunk), sizeof(int32_t) * K * E, st, g, choice, ord, s.hist,
                                                                           flags);
    launch_pdl(assign_scan_kernel, dim3((int)ceil_div(E, 128)), dim3(128), 0, st, g, s.hist, s.base, s.gkept, kept);
    launch_pdl(assign_rank_kernel, dim3(nchunks), dim3(kChunk), sizeof(int32_t) * 32 * E, st, 
        g, choice, ord, s.base, s.gkept, cap_pad, slot, pos, row_src);
}

size_t assign_scratch_ints(int64_t T, int E, int K, int G) {
    const int64_t chunks = (int64_t)G * ceil_div(ceil_div(T, G), kChunk) + G;
    return (size_t)(2 * chunks * K * E + 2 * (int64_t)G * E + 64);
}

// ---------------------------------------------------------------------------
// Backward of the routing weights + balance loss + softmax, one warp per
// token (the closures of ops.cpp:250-281, 552-558, 528-537, 579-585, 329-343):
//   dw_k = <dy[t], O[row_k]> for kept routes (routing.cpp:337-342)
//   top-1: dp0 = E * dw0;  top-2: dp_k = dw_k/S - (dw0 p0 + dw1 p1)/S^2
//   dP[t,e] = daux * fcoef[e] + sum_k [e == c_k] dp_k
//   dL[t,e] = P[t,e] * (dP[t,e] - <dP[t], P[t]>)
// ---------------------------------------------------------------------------
template <class TIO, int V>
__global__ void __launch_bounds__(256)
router_bwd_kernel(int64_t T, int d, int E, int K, const TIO* __restrict__ dy,
                  const TIO* __restrict__ O, int cap_pad, const int32_t* __restrict__ choice,
                  const int32_t* __restrict__ pos, const float* __restrict__ gate_prob,
                  const float* __restrict__ probs, const float* __restrict__ fcoef, float daux,
                  float* __restrict__ dL, float* __restrict__ dLr) {
    pdl_wait();
    pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t = (int64_t)blockIdx.x * 8 + warp;
    if (t >= T) return;
    float dw[2] = {0.f, 0.f};
    #pragma unroll
    for (int k = 0; k < 2; ++k) {  // K <= 2
        if (k >= K) break;
        const int32_t p = pos[t * K + k];
        if (p < 0) continue;
        const int64_t row = (int64_t)choice[t * K + k] * cap_pad + p;
        float acc = 0.f;
#pragma unroll 4
        for (int j = lane * V; j < d; j += 32 * V) {
            float a[V], b[V];
            load_f<TIO, V>(dy + t * d + j, a);
            load_f<TIO, V>(O + row * d + j, b);
#pragma unroll
            for (int q = 0; q < V; ++q) acc = fmaf(a[q], b[q], acc);
        }
        dw[k] = warp_sum(acc);
    }
    float dp[2];
    if (K == 1) {
        dp[0] = (float)E * dw[0];
        dp[1] = 0.f;
    } else {
        const float p0 = gate_prob[t * 2], p1 = gate_prob[t * 2 + 1];
        const float S = p0 + p1;
        const float ds = -(dw[0] * p0 + dw[1] * p1) / (S * S);
        dp[0] = dw[0] / S + ds;
        dp[1] = dw[1] / S + ds;
    }
    const int c0 = choice[t * K];
    const int c1 = K == 2 ? choice[t * K + 1] : -1;
    float dot = 0.f;
    for (int e = lane; e < E; e += 32) {
        float g = daux * fcoef[e];
        if (e == c0) g += dp[0];
        if (e == c1) g += dp[1];
        dot = fmaf(g, probs[t * E + e], dot);
    }
    dot = warp_sum(dot);
    for (int e = lane; e < E; e += 32) {
        float g = daux * fcoef[e];
        if (e == c0) g += dp[0];
        if (e == c1) g += dp[1];
        const float v = probs[t * E + e] * (g - dot);
        dL[t * E + e] = v;
        if (dLr) dLr[t * E + e] = tf32_rna_dev(v);
    }
}

// The same with the combine backward folded in (single-rank layers): the warp
// that reads dy[t] for <dy, O[row_k]> also writes dO[row_k] = w_k dy[t]
// (permute.cu combine_bwd_gather_kernel), so dy is read once and the two
// passes become one.  Blocks past the token range zero the expert tails
// [kept[e], roundup(kept[e], 128)) that the tensor-core tiles read.  The dot
// products accumulate in the same order as router_bwd_kernel.
template <class TIO, int V>
__global__ void __launch_bounds__(256, 4)
router_combine_bwd_kernel(int64_t T, int d, int E, int K, const TIO* __restrict__ dy,
                          const TIO* __restrict__ O, int cap_pad, const int32_t* __restrict__ choice,
                          const int32_t* __restrict__ pos, const float* __restrict__ gate_prob,
                          const float* __restrict__ probs, const float* __restrict__ fcoef, float daux,
                          const float* __restrict__ w, const int32_t* __restrict__ kept,
                          TIO* __restrict__ dO, float* __restrict__ dL, float* __restrict__ dLr, RowDst rd) {
    pdl_wait();
    pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t tok_blocks = (T + 7) / 8;
    // dO row (e, p): local [E][cap_pad], or under EP straight in expert e's owner
    auto drow = [&](int e, int64_t p) -> TIO* {
        return rd.ep > 1 ? static_cast<TIO*>(rd.p[e / rd.El]) + ((int64_t)(e % rd.El) * cap_pad + p) * d
                         : dO + ((int64_t)e * cap_pad + p) * d;
    };
    if ((int64_t)blockIdx.x >= tok_blocks) {  // expert tails
        const int64_t q = ((int64_t)blockIdx.x - tok_blocks) * 8 + warp;
        const int e = (int)(q / kRowAlign);
        if (e >= E) return;
        const int n = kept[e];
        const int64_t p = n + q % kRowAlign;
        if (p >= round_up_dev(n, kRowAlign)) return;
        TIO* dst = drow(e, p);
        for (int64_t j = (int64_t)lane * V; j < d; j += 32 * V) zero_vec<TIO, V>(dst + j);
        return;
    }
    const int64_t t = (int64_t)blockIdx.x * 8 + warp;
    if (t >= T) return;
    int64_t row[2] = {-1, -1};
    TIO* dOr_[2] = {nullptr, nullptr};
    float wk[2] = {0.f, 0.f};
#pragma unroll
    for (int k = 0; k < 2; ++k) {  // K <= 2
        if (k >= K) break;
        const int32_t p = pos[t * K + k];
        if (p < 0) continue;
        const int32_t ce = choice[t * K + k];
        row[k] = (int64_t)ce * cap_pad + p;
        dOr_[k] = drow(ce, p);
        wk[k] = w[t * K + k];
    }
    // the softmax-backward operands, loaded ahead of the row traffic (E <= 64)
    float pe[2], fe[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int e = lane + 32 * i;
        pe[i] = e < E ? __ldg(probs + t * E + e) : 0.f;
        fe[i] = e < E ? __ldg(fcoef + e) : 0.f;
    }
    float acc[2] = {0.f, 0.f};
    const TIO* dyt = dy + t * d;
    if constexpr (V * sizeof(TIO) == 16) {
        // raw 16-byte vectors in registers (kU per operand in flight per lane)
        constexpr int kU = 4;
        for (int j0 = lane * V; j0 < d; j0 += 32 * V * kU) {
            Vec16<TIO> a[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u)
                if (j0 + u * 32 * V < d) a[u].u = __ldg(reinterpret_cast<const uint4*>(dyt + j0 + u * 32 * V));
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                if (row[k] < 0) continue;
                const TIO* Ok = O + row[k] * d;
                TIO* dOk = dOr_[k];
                Vec16<TIO> b[kU];
#pragma unroll
                for (int u = 0; u < kU; ++u)
                    if (j0 + u * 32 * V < d) b[u].u = __ldg(reinterpret_cast<const uint4*>(Ok + j0 + u * 32 * V));
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    if (j0 + u * 32 * V >= d) continue;
                    Vec16<TIO> o;
#pragma unroll
                    for (int q = 0; q < V; ++q) {
                        const float av = to_f(a[u].e[q]);
                        acc[k] = fmaf(av, to_f(b[u].e[q]), acc[k]);
                        o.e[q] = from_f<TIO>(av * wk[k]);
                    }
                    *reinterpret_cast<uint4*>(dOk + j0 + u * 32 * V) = o.u;
                }
            }
        }
    } else {
        for (int j = lane * V; j < d; j += 32 * V) {
            float a[V];
            load_f<TIO, V>(dyt + j, a);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                if (row[k] < 0) continue;
                float b[V], v[V];
                load_f<TIO, V>(O + row[k] * d + j, b);
#pragma unroll
                for (int q = 0; q < V; ++q) {
                    acc[k] = fmaf(a[q], b[q], acc[k]);
                    v[q] = a[q] * wk[k];
                }
                store_f<TIO, V>(dOr_[k] + j, v);
            }
        }
    }
    float dw[2];
    dw[0] = row[0] >= 0 ? warp_sum(acc[0]) : 0.f;
    dw[1] = row[1] >= 0 ? warp_sum(acc[1]) : 0.f;
    float dp[2];
    if (K == 1) {
        dp[0] = (float)E * dw[0];
        dp[1] = 0.f;
    } else {
        const float p0 = gate_prob[t * 2], p1 = gate_prob[t * 2 + 1];
        const float S = p0 + p1;
        const float ds = -(dw[0] * p0 + dw[1] * p1) / (S * S);
        dp[0] = dw[0] / S + ds;
        dp[1] = dw[1] / S + ds;
    }
    const int c0 = choice[t * K];
    const int c1 = K == 2 ? choice[t * K + 1] : -1;
    float g[2];
    float dot = 0.f;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int e = lane + 32 * i;
        g[i] = daux * fe[i];
        if (e == c0) g[i] += dp[0];
        if (e == c1) g[i] += dp[1];
        if (e < E) dot = fmaf(g[i], pe[i], dot);
    }
    dot = warp_sum(dot);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int e = lane + 32 * i;
        if (e < E) {
            const float v = pe[i] * (g[i] - dot);
            dL[t * E + e] = v;
            if (dLr) dLr[t * E + e] = tf32_rna_dev(v);
        }
    }
}

template <class TIO>
void launch_router_combine_bwd(int64_t T, int d, int E, int K, const TIO* dy, const TIO* O, int cap_pad,
                               const int32_t* choice, const int32_t* pos, const float* gate_prob,
                               const float* probs, const float* fcoef, float daux, const float* w,
                               const int32_t* kept, TIO* dO, float* dL, cudaStream_t st, float* dLr,
                               const RowDst* rd) {
    RowDst r0{};
    const RowDst& rdv = rd ? *rd : r0;
    if (E > 64) throw Status(6, "router_combine_bwd: E <= 64");
    const unsigned grid = (unsigned)(ceil_div(T, (int64_t)8) + ceil_div((int64_t)E * kRowAlign, (int64_t)8));
    if (vec_width<TIO>(d) > 1)
        launch_pdl(router_combine_bwd_kernel<TIO, 16 / sizeof(TIO)>, dim3(grid), dim3(256), 0, st, T, d, E, K,
                   dy, O, cap_pad, choice, pos, gate_prob, probs, fcoef, daux, w, kept, dO, dL, dLr, rdv);
    else
        launch_pdl(router_combine_bwd_kernel<TIO, 1>, dim3(grid), dim3(256), 0, st, T, d, E, K, dy, O, cap_pad,
                   choice, pos, gate_prob, probs, fcoef, daux, w, kept, dO, dL, dLr, rdv);
}
template void launch_router_combine_bwd<float>(int64_t, int, int, int, const float*, const float*, int,
                                               const int32_t*, const int32_t*, const float*, const float*,
                                               const float*, float, const float*, const int32_t*, float*,
                                               float*, cudaStream_t, float*, const RowDst*);
template void launch_router_combine_bwd<__nv_bfloat16>(int64_t, int, int, int, const __nv_bfloat16*,
                                                       const __nv_bfloat16*, int, const int32_t*,
                                                       const int32_t*, const float*, const float*,
                                                       const float*, float, const float*, const int32_t*,
                                                       __nv_bfloat16*, float*, cudaStream_t, float*,
                                                       const RowDst*);

template <class TIO>
void launch_router_bwd(int64_t T, int d, int E, int K, const TIO* dy, const TIO* O, int cap_pad,
                       const int32_t* choice, const int32_t* pos, const float* gate_prob,
                       const float* probs, const float* fcoef, float daux, float* dL,
                       cudaStream_t st, float* dLr) {
    if (vec_width<TIO>(d) > 1)
        launch_pdl(router_bwd_kernel<TIO, 16 / sizeof(TIO)>, dim3((int)ceil_div(T, 8)), dim3(256), 0, st, 
            T, d, E, K, dy, O, cap_pad, choice, pos, gate_prob, probs, fcoef, daux, dL, dLr);
    else
        launch_pdl(router_bwd_kernel<TIO, 1>, dim3((int)ceil_div(T, 8)), dim3(256), 0, st, 
            T, d, E, K, dy, O, cap_pad, choice, pos, gate_prob, probs, fcoef, daux, dL, dLr);
}

template void launch_router_bwd<float>(int64_t, int, int, int, const float*, const float*, int,
                                       const int32_t*, const int32_t*, const float*, const float*,
                                       const float*, float, float*, cudaStream_t, float*);
template void launch_router_bwd<__nv_bfloat16>(int64_t, int, int, int, const __nv_bfloat16*,
                                               const __nv_bfloat16*, int, const int32_t*,
                                               const int32_t*, const float*, const float*,
                                               const float*, float, float*, cudaStream_t, float*);

}  // namespace moe

namespace moe {

// balance_loss over explicit probabilities (routing.cpp:348-374): per-CTA
// column sums / first-choice counts / row-sum check, then the same finalize.
__global__ void __launch_bounds__(256)
balance_partials_kernel(const float* __restrict__ probs, int64_t T, int E, int K,
                        const int32_t* __restrict__ eid, float* __restrict__ colsum_part,
                        int32_t* __restrict__ count_part, uint32_t* __restrict__ flags) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ float sm[];
    float* s_col = sm;
    int32_t* s_cnt = reinterpret_cast<int32_t*>(sm + 8 * E);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 8 * E; i += blockDim.x) s_col[i] = 0.f;
    for (int i = threadIdx.x; i < E; i += blockDim.x) s_cnt[i] = 0;
    __syncthreads();
    uint32_t flag = 0;
    const int64_t t0 = (int64_t)blockIdx.x * kRowsPerPart;
    for (int64_t t = t0 + warp; t < min(T, t0 + kRowsPerPart); t += 8) {
        float s = 0.f;
        for (int e = lane; e < E; e += 32) {
            const float p = probs[t * E + e];
            s_col[warp * E + e] += p;
            s += p;
        }
        s = warp_sum(s);
        if (lane == 0) {
            const int c = eid[t * K];
            if (c >= 0 && c < E) atomicAdd(&s_cnt[c], 1); else flag |= MOE_FLAG_CHOICE_RANGE_DEV;
            if (!(fabsf(s - 1.0f) <= kProbRowTol)) flag |= MOE_FLAG_PROB_ROWS_DEV;
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        float acc = 0.f;
        for (int w = 0; w < 8; ++w) acc += s_col[w * E + e];
        colsum_part[(int64_t)blockIdx.x * E + e] = acc;
        count_part[(int64_t)blockIdx.x * E + e] = s_cnt[e];
    }
    if (lane == 0 && flag) atomicOr(flags, flag);
}

void launch_balance_from_probs(const float* probs, int64_t T, int E, int K,
                               const int32_t* expert_id, double alpha, float* loss,
                               float* colsum_part, int32_t* count_part, uint32_t* flags,
                               double* term, unsigned* done, cudaStream_t st) {
    const int nparts = softmax_parts(T);
    launch_pdl(balance_partials_kernel, dim3(nparts), dim3(256), sizeof(float) * 8 * E + sizeof(int32_t) * E, st, 
        probs, T, E, K, expert_id, colsum_part, count_part, flags);
    launch_balance_finalize(colsum_part, count_part, nparts, T, E, alpha, loss, nullptr, nullptr,
                            term, done, st);
}

}  // namespace moe
