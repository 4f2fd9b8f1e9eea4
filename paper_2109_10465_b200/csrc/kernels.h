// kernels.h — launch interfaces of the B200 MoE layer kernels (internal).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace moe {

// device flag bits (mirror MOE_FLAG_* in include/moe_b200.h)
constexpr uint32_t MOE_FLAG_NONFINITE_DEV = 0x1u;
constexpr uint32_t MOE_FLAG_PROB_ROWS_DEV = 0x2u;
constexpr uint32_t MOE_FLAG_CHOICE_RANGE_DEV = 0x4u;
constexpr uint32_t MOE_FLAG_UNIFORM_SHAPE_DEV = 0x8u;
constexpr uint32_t MOE_FLAG_RTS_OVERFLOW_DEV = 0x10u;
// fp32 probabilities: |sum_e P - 1| bound used in place of the reference's
// f64 1e-9 (routing.cpp:360-361).
constexpr float kProbRowTol = 1e-4f;

// ---- router.cu ------------------------------------------------------------
int softmax_parts(int64_t T);
// logits may be `nsplit` split-K partial arrays [nsplit][T][E], summed in
// fixed order before the softmax.
void launch_softmax_topk(const float* logits, int nsplit, int64_t T, int E, int K, float* probs,
                         int32_t* choice, float* gate_prob, float* colsum_part,
                         int32_t* count_part, uint32_t* flags, cudaStream_t st);
constexpr int kMaxGateSplits = 8;
int gate_logit_splits(int64_t T, int d, int E);
void launch_balance_finalize(const float* colsum_part, const int32_t* count_part, int nparts,
                             int64_t T, int E, double alpha, float* aux, float* fcoef,
                             int32_t* counts, double* term, unsigned* done, cudaStream_t st);

struct AssignScratch {
    int32_t* hist;   // [chunks][K][E]
    int32_t* base;   // [chunks][K][E]
    int32_t* gkept;  // [G][2][E]
    int max_chunks;
    int max_groups;
};
size_t assign_scratch_ints(int64_t T, int E, int K, int G);
void launch_assign(int64_t T, int E, int K, int cap, int mode, int G, const int32_t* choice,
                   const uint32_t* ord, int cap_pad, AssignScratch& s, int32_t* slot, int32_t* pos,
                   int32_t* row_src, int32_t* kept, uint32_t* flags, cudaStream_t st);

template <class TIO>
void launch_router_bwd(int64_t T, int d, int E, int K, const TIO* dy, const TIO* O, int cap_pad,
                       const int32_t* choice, const int32_t* pos, const float* gate_prob,
                       const float* probs, const float* fcoef, float daux, float* dL,
                       cudaStream_t st, float* dLr = nullptr);

// Row destinations under expert parallelism: p[o] = rank o's receive buffer
// at this rank's slot (local buffer for o == rank); expert e's rows go to
// p[e / El] at local expert e % El.  ep <= 1: the local [E][cap_pad] buffer.
struct RowDst {
    void* p[8];
    int El;
    int ep;
};
// router_bwd with the combine backward (dO rows = w dy[t], expert tails
// zeroed) folded in: one pass over dy for single-rank layers.
template <class TIO>
void launch_router_combine_bwd(int64_t T, int d, int E, int K, const TIO* dy, const TIO* O, int cap_pad,
                               const int32_t* choice, const int32_t* pos, const float* gate_prob,
                               const float* probs, const float* fcoef, float daux, const float* w,
                               const int32_t* kept, TIO* dO, float* dL, cudaStream_t st,
                               float* dLr = nullptr, const RowDst* rd = nullptr);

// ---- rng.cu ---------------------------------------------------------------
// Jitter noise n[i] = lo + (hi-lo) * ((mt() >> 11) * 2^-53) for i in [0, count)
// of the mt19937_64 stream seeded with `seed` (routing.cpp:62-70), generated
// on the device with jump-ahead (see rng.cu).
struct MtJumpTable;
void launch_jitter_noise(const MtJumpTable* tab, uint64_t seed, int64_t count, double eps,
                         float* noise, cudaStream_t st);

// ---- permute.cu -----------------------------------------------------------
// Buffer geometry: nseg = ep * E_local segments; segment (r, le) holds rows
// [(r*E_local + le) * cap_pad, ... + cap_pad) of the expert-input buffer,
// the first counts[r*E_local+le] of which are occupied.
template <class TIO>
void launch_dispatch_gather(const TIO* x, int64_t d, int E, int K, int cap_pad,
                            const int32_t* row_src, const int32_t* kept, TIO* buf,
                            uint32_t* flags, cudaStream_t st, const RowDst* rd = nullptr);
template <class TIO>
void launch_combine(const TIO* O, int64_t T, int64_t d, int E, int K, int cap_pad,
                    const int32_t* choice, const int32_t* pos, const float* w,
                    const TIO* residual, TIO* y, uint32_t* flags, cudaStream_t st);
template <class TIO>
void launch_combine_bwd_gather(const TIO* dy, int64_t d, int E, int K, int cap_pad,
                               const int32_t* row_src, const int32_t* kept, const float* w,
                               TIO* dO, cudaStream_t st);
// dx[t] = dxg[t] * noise[t] + sum_k dX[row_k] + (residual is x && none kept ? dy[t] : 0)
// and dres[t] = none kept ? dy[t] : 0 when residual was explicit.
template <class TIO>
void launch_dx_assemble(int64_t T, int64_t d, int E, int K, int cap_pad, const float* dxg,
                        const float* noise, const TIO* dX, const int32_t* choice,
                        const int32_t* pos, const TIO* dy, bool residual_is_x, TIO* dx,
                        TIO* dres, cudaStream_t st);
void launch_combine_weights(int64_t T, int E, int K, const float* gate_prob, float* w,
                            cudaStream_t st);
// utilization / drop-position statistics of a decision (int64 accumulators)
void launch_decision_stats(int64_t T, int E, int K, const int32_t* choice, const int32_t* pos,
                           int64_t* util, int64_t* hist, cudaStream_t st);
// db[g][n] = sum over the group's occupied rows of src[row][n]
template <class TIO>
void launch_colsum_groups(const TIO* src, int64_t N, int ep, int El, int cap_pad,
                          const int32_t* counts, float* db, cudaStream_t st);
// db[g][n] = sum over the group's computed 32-row blocks of part[blk][n]
// (the fused GEMM-epilogue column sums of RowGemmArgs::colsum), fixed order
void launch_colsum_parts(const float* part, int64_t N, int ep, int El, int cap_pad,
                         const int32_t* counts, float* db, cudaStream_t st);
// reference-layout per-stage dispatch / combine (routing.cpp:208-298)
template <class TIO>
void launch_dispatch_ref(const TIO* x, int64_t T, int64_t d, int E, int K, int cap,
                         const int32_t* expert_id, const int32_t* slot, TIO* buf, uint8_t* occ,
                         cudaStream_t st);
template <class TIO>
void launch_combine_ref(const TIO* O, int64_t T, int64_t d, int E, int K, int cap,
                        const int32_t* expert_id, const int32_t* slot, const float* w,
                        const TIO* residual, TIO* y, cudaStream_t st);
void launch_check_finite_f32(const float* p, int64_t n, uint32_t* flags, cudaStream_t st);

// ---- gemm_simt.cu (fp32 SIMT; the parity path and the gate GEMMs) ----------
// Dense C[M,N] = sum_k A(m,k) * B(k,n), A(m,k) = A[m*lda_m + k*lda_k] * (S ? S[same] : 1),
// B(k,n) = B[k*ldb_k + n*ldb_n].  split_k > 1 writes partial sums to
// C + s*M*N (caller reduces with launch_splitk_reduce).
template <class TA>
void launch_gemm_dense(const TA* A, int64_t lda_m, int64_t lda_k, const float* S,
                       const float* B, int64_t ldb_k, int64_t ldb_n, float* C, int64_t M,
                       int64_t N, int64_t K, int split_k, cudaStream_t st);
void launch_splitk_reduce(const float* part, int split_k, int64_t MN, float* out,
                          cudaStream_t st);

enum EpiKind { EPI_BIAS_RELU = 0, EPI_BIAS = 1, EPI_RELU_MASK = 2, EPI_NONE = 3 };

// Expert GEMM over buffer rows (fwd1, fwd2, dgrad2, dgrad1):
//   C[row, n] = epi( sum_k A[row, k] * W_le(k, n) )
// rows of segment (r, le) are [(r*El+le)*cap_pad, + counts[r*El+le]);
// W_le(k,n) = W[le*K*N + k*N + n] if w_nmajor else W[le*N*K + n*K + k].
// Rows in [count, roundup(count,128)) of each segment are written as zero.
struct RowGemmArgs {
    const void* A;
    const void* W;
    void* C;
    const float* bias;   // [El][N] (EPI_BIAS*)
    const void* mask;    // H buffer for EPI_RELU_MASK (same layout as C)
    const int32_t* counts;
    int64_t N, K;
    int ep, El, cap_pad;
    bool w_nmajor;
    int epi;
    // optional (tensor-core path, EPI_RELU_MASK): per-32-row-block column sums
    // of the stored C, [rows/32][N]; reduce with launch_colsum_parts
    float* colsum = nullptr;
    // optional (tensor-core path, expert parallelism): store each origin rank
    // r's rows straight into c_peer[r] (rank r's receive buffer slice for this
    // rank, [El * cap_pad][N], NVLink-mapped), row (seg % El) * cap_pad + m,
    // instead of C — the combine exchange's copy folded into the epilogue
    void* const* c_peer = nullptr;
    // SMs left free for a co-running kernel (the jitter prefetch); the
    // persistent grid uses the rest
    int sm_reserve = 0;
    // optional (tensor-core path): the ReLU mask as bits, [rows][N/64] words —
    // written by EPI_BIAS_RELU (bit j of word (row, c) = stored bf16 H > 0),
    // read by EPI_RELU_MASK instead of the bf16 H (16x fewer bytes)
    uint64_t* relu_bits = nullptr;
};
template <class T>
void launch_row_gemm_simt(const RowGemmArgs& a, cudaStream_t st);

// Expert weight-gradient GEMM: Cg[m, n] = sum_{r, i < count(r,g)} A[row, m] * B[row, n]
struct WgradGemmArgs {
    const void* A;   // [rows][M]
    const void* B;   // [rows][N]
    void* C;         // [El][M][N]
    const int32_t* counts;
    int64_t M, N;
    int ep, El, cap_pad;
    int sm_reserve = 0;  // as RowGemmArgs::sm_reserve
    // output mode: bit 0 = accumulate into C (the tape's +=, tensor.cpp:31-36),
    // bit 1 = C is fp32 (fp32 weight gradients of a bf16 layer)
    int c_mode = 0;
};
template <class T>
void launch_wgrad_gemm_simt(const WgradGemmArgs& a, cudaStream_t st);

}  // namespace moe

namespace moe {
// rng.cu: device mt19937_64 jitter stream; returns false if the device
// generator cannot serve this request (caller then uploads the host stream).
// max_ctas: the stream is cut into at most that many chunks, one CTA (one SM)
// each (a generator that co-runs with kernels owning the other SMs)
bool launch_jitter_noise_device(uint64_t seed, int64_t count, double eps, float* noise,
                                cudaStream_t st, int max_ctas = 148);
// router.cu: balance_loss from explicit probabilities (per-stage API)
void launch_balance_from_probs(const float* probs, int64_t T, int E, int K,
                               const int32_t* expert_id, double alpha, float* loss,
                               float* colsum_part, int32_t* count_part, uint32_t* flags,
                               double* term, unsigned* done, cudaStream_t st);
}  // namespace moe

namespace moe {
// gate.cu: register-tiled gate GEMMs (require gate_fast_ok(d, E))
bool gate_fast_ok(int d, int E);
template <class TX>
void launch_gate_logits(const TX* x, const float* noise, const float* wg, float* logits,
                        int64_t T, int d, int E, int splits, cudaStream_t st);
template <class TIO>
void launch_gate_dx(int64_t T, int d, int E, int K, int cap_pad, const float* dL, const float* wg,
                    const float* noise, const TIO* dX, const int32_t* choice, const int32_t* pos,
                    const TIO* dy, bool residual_is_x, TIO* dx, TIO* dres, cudaStream_t st);
template <class TX>
void launch_gate_dw(const TX* x, const float* noise, const float* dL, float* part, int64_t T,
                    int d, int E, int splits, cudaStream_t st);
}  // namespace moe

namespace moe {
constexpr int kMaxCopies = 16;
struct PeerCopyJobs {
    const void* src[kMaxCopies];
    void* dst[kMaxCopies];
    int64_t bytes[kMaxCopies];
    int n;
};
void launch_peer_copy(const PeerCopyJobs& jobs, cudaStream_t st);
struct PeerFlags {
    unsigned long long* f[8];  // each rank's flag array, mapped into this process
};
// Per-rank token-count agreement carried by an exchange barrier (tokens < 0:
// no check).  On mismatch: flags |= MOE_FLAG_UNIFORM_SHAPE, counts[0..n) = 0.
struct ShapeCheck {
    long long tokens;
    uint32_t* flags;
    int32_t* counts;
    int ncounts;
};
void launch_ipc_barrier(const PeerFlags& peers, const unsigned long long* mine, int rank, int ep,
                        unsigned long long epoch, cudaStream_t st, const ShapeCheck* sc = nullptr);
void launch_fill_i64(long long* p, long long v, cudaStream_t st);
void launch_ep_shape_check(const long long* all_t, int ep, const ShapeCheck& sc, cudaStream_t st);
// out = sum over ranks of src[r] (fixed rank order), n % 4 == 0
void launch_sum_ranks(const float* const* srcs, int ep, int64_t n, float* out, cudaStream_t st);

// gate2.cu: larger-tile gate GEMMs (require gate2_ok(d, E))
bool gate2_ok(int d, int E);
int gate2_logit_splits(int64_t T, int d, int E);
template <class TX>
void launch_gate2_logits(const TX* x, const float* noise, const float* wg, float* logits, int64_t T,
                         int d, int E, int splits, cudaStream_t st);
void launch_gate2_transpose(const float* wg, float* wgt, int d, int E, cudaStream_t st);
template <class TIO>
void launch_gate2_dx(int64_t T, int d, int E, int K, int cap_pad, const float* dL, const float* wgt,
                     const float* noise, const TIO* dX, const int32_t* choice, const int32_t* pos,
                     const TIO* dy, bool residual_is_x, TIO* dx, TIO* dres, cudaStream_t st);
// gate_tc.cu: tensor-core (kind::tf32) gate GEMMs for the bf16 path
bool gate_tc_ok(int d, int E);
int gate_tc_logit_splits(int64_t T, int d);
// wgt = Wg^T [E][d] (launch_gate2_transpose)
template <class TX>
void launch_gate_tc_logits(const TX* x, const float* noise, const float* wgt, float* logits, int64_t T,
                           int d, int E, int splits, cudaStream_t st);
template <class TX>
void launch_gate_tc_dw(const TX* x, const float* noise, const float* dL, float* part, int64_t T, int d,
                       int E, int splits, cudaStream_t st);
template <class TIO>
void launch_gate_tc_dx(int64_t T, int d, int E, int K, int cap_pad, const float* dL, const float* wg,
                       const float* noise, const TIO* dX, const int32_t* choice, const int32_t* pos,
                       const TIO* dy, bool residual_is_x, TIO* dx, TIO* dres, cudaStream_t st);
// dxg = (dL Wg^T) * noise in fp32 (noise may be null)
void launch_gate2_dxg(int64_t T, int d, int E, const float* dL, const float* wgt, const float* noise,
                      float* dxg, cudaStream_t st);
}  // namespace moe

namespace moe {
// optim.cu: AdamOptimizer::step on the device (optim.cpp:21-57)
void launch_grad_sqnorm(const void* g, int64_t n, bool bf16, double* acc, cudaStream_t st);
void launch_clip_scale(const double* sq, double clip, double* scale, cudaStream_t st);
void launch_adam(float* theta, float* m, float* v, const void* g, int64_t n, bool g_bf16,
                 __nv_bfloat16* shadow, const double* scale, double lr, double b1, double b2,
                 double eps, int64_t step, cudaStream_t st);
}  // namespace moe

namespace moe {
// permute.cu: f64 checkpoint record -> fp32 / bf16 device tensor
void launch_convert_f64(const double* src, int64_t n, bool bf16, void* dst, cudaStream_t st);
}  // namespace moe

namespace moe {
// f64_layer.cu: the reference-precision (float64) path, see the file header
void launch_mt64_raw_device(uint64_t seed, int64_t count, uint64_t* out, cudaStream_t st);
void launch_f64_noise(uint64_t* buf, int64_t n, double lo, double hi, cudaStream_t st);
void launch_f64_gate(const double* x, const double* noise, const double* gw, double* L, double* P, int64_t T,
                     int d, int E, int K, int32_t* choice, double* gp, uint32_t* flags, cudaStream_t st);
void launch_f64_balance(const double* P, const int32_t* choice, int64_t T, int E, int K, double alpha,
                        double* aux, double* fval, cudaStream_t st);
void launch_f64_weights(const double* gp, int64_t T, int E, int K, double* w, cudaStream_t st);
void launch_f64_dispatch(const double* x, int64_t d, int E, int K, int cap_pad, const int32_t* row_src,
                         const int32_t* kept, double* X, cudaStream_t st);
void launch_f64_seg_gemm(const double* A, const double* W, double* C, const double* bias, const double* M,
                         const int32_t* kept, int E, int cap_pad, int64_t K, int64_t N, bool nmajor, int epi,
                         cudaStream_t st);
void launch_f64_seg_wgrad(const double* A, const double* B, double* C, const int32_t* kept, int E, int cap_pad,
                          int64_t M, int64_t N, bool accumulate, cudaStream_t st);
void launch_f64_combine(const double* O, const double* res, int64_t T, int64_t d, int K, int cap_pad,
                        const int32_t* choice, const int32_t* pos, const double* w, double* y,
                        uint32_t* flags, cudaStream_t st);
void launch_f64_combine_bwd(const double* dy, const double* O, int64_t T, int64_t d, int K, int cap_pad,
                            const int32_t* choice, const int32_t* pos, const double* w, double* dO, double* dw,
                            cudaStream_t st);
void launch_f64_router_bwd(const double* P, const double* gp, const double* dw, const int32_t* choice,
                           const double* fval, double daux, int64_t T, int E, int K, double* dL,
                           cudaStream_t st);
void launch_f64_gate_dw(const double* x, const double* noise, const double* dL, double* dW, int64_t T, int d,
                        int E, bool accumulate, cudaStream_t st);
void launch_f64_dx(const double* dL, const double* gw, const double* noise, const double* dX, const double* dy,
                   int64_t T, int d, int E, int K, int cap_pad, const int32_t* choice, const int32_t* pos,
                   bool residual_is_x, double* dx, double* dres, bool accumulate, cudaStream_t st);
void launch_f64_acc_copy(const double* src, double* dst, int64_t n, bool accumulate, cudaStream_t st);
}  // namespace moe

namespace moe {
// gate_fused.cu: logits + softmax + top-k + balance partials + balance finalize
// in one cluster kernel (bf16 path, E in {8, 16, 32, 64})
bool gate_fused_ok(int d, int E);
int gate_fused_parts(int64_t T);
// wsplit [2][EP][d]: tf32 hi / lo halves of Wg^T, EP = max(E, 16) rows (zero-padded)
size_t gate_split_floats(int d, int E);
void launch_gate_split(const float* wg, float* wsplit, int d, int E, cudaStream_t st);
int gate_fused_stamps(unsigned long long* host, int ncta);  // debug (MOE_B200_GATE_PROBE=8)
// writes P, the decision and per-64-token balance partials [gate_fused_parts][E]
// (finalize with launch_balance_finalize)
void launch_gate_fused(const __nv_bfloat16* x, const float* noise, const float* wsplit, int64_t T, int d, int K,
                       int E, float* probs, int32_t* choice, float* gate_prob, float* colsum_part,
                       int32_t* count_part, uint32_t* flags, cudaStream_t st);
}  // namespace moe

namespace moe {
// gate_bwd.cu: dWg partials [splits][d][E] = (x*noise)^T dL on the tensor
// cores, TMA-fed with MN-major operands (bf16 path, E == 64, d % 128 == 0)
bool gate_dw_tma_ok(int d, int E);
void launch_gate_dw_tma(const __nv_bfloat16* x, const float* noise, const float* dL, float* part, int64_t T, int d,
                        int splits, cudaStream_t st);
// dx = (dLr WgR^T) * noise + dispatch-backward rows (+ dy / dres), persistent
// TMA-fed tcgen05 kernel; dLr / WgR are the tf32-rounded dL / Wg
bool gate_dx_tma_ok(int d, int E, int K);
void launch_gate_round_wg(const float* wg, float* wgr, int d, int E, cudaStream_t st);
void launch_gate_dx_tma(int64_t T, int d, int K, int cap_pad, const float* dLr, const float* wgr, const float* noise,
                        const __nv_bfloat16* dX, const int32_t* choice, const int32_t* pos, const __nv_bfloat16* dy,
                        bool residual_is_x, __nv_bfloat16* dx, __nv_bfloat16* dres, cudaStream_t st);
}  // namespace moe

namespace moe {
// rts.cu: Rng(seed).permutation(n) on the device (the RTS priority order)
size_t rts_scratch_bytes(int64_t n);
void launch_rts_order(uint64_t seed, int64_t n, void* scratch, uint32_t* perm, uint32_t* layer_flags,
                      cudaStream_t st);
}  // namespace moe

namespace moe {
// dst[i] += src[i] (fp32 math; dst and src both bf16 or both fp32)
void launch_add_into(void* dst, const void* src, int64_t n, bool bf16, cudaStream_t st);
}  // namespace moe
