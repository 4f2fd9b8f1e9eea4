/*
 * moe_b200.h — C ABI of the B200-native MoE layer (libmoe_b200.so).
 *
 * Drop-in boundary for the reference's MoE-layer operator API
 * (/root/reference/proj/core/include/moeforge/routing.hpp, parallel.hpp).
 * The reference has no FFI of its own: its "operator API" is that C++ header,
 * linked statically.  This ABI exposes the same operations with plain
 * pointers and sizes (no C++ or torch types) so C++, Python (ctypes) or any
 * other FFI can bind it; include/moe_b200.hpp layers the reference's C++
 * names (RouterConfig, RoutingDecision, moe_layer_forward, ...) on top.
 *
 * Conventions
 *  - Every tensor argument is a DEVICE pointer (caller-owned; the library
 *    never frees caller memory) unless the name ends in _host.
 *  - Row-major layouts identical to the reference:
 *      x, y, residual, dy, dx      [T, d_model]
 *      gate_w                      [d_model, E]            (routing.hpp:126)
 *      w1 [E_local, d_model, d_ff], b1 [E_local, d_ff]      (model.cpp:77-83, ExpertFfn)
 *      w2 [E_local, d_ff, d_model], b2 [E_local, d_model]
 *      decisions: entry (t, k) at index t * top_k + k      (routing.hpp:36-37)
 *  - dtype MOE_F32: activations and expert weights are float32 (parity path,
 *    1e-5 relative).  MOE_BF16: activations, expert weights and their grads
 *    are bfloat16 with fp32 accumulation (tcgen05 path).  gate_w, biases,
 *    gate probabilities and their grads are always float32.
 *  - Exceptions never cross the ABI: each call returns a moe_status that maps
 *    1:1 to the reference exception types (common.hpp:10-35); the text is
 *    available from moe_last_error().  Device-side conditions (non-finite
 *    values, probability rows not summing to one) are latched in a device
 *    flag word and reported by moe_check() (which synchronises the stream).
 *  - One handle = one CUDA stream = one layer's saved context; a handle is
 *    not re-entrant, distinct handles are thread-safe (SPEC threading model,
 *    tensor.hpp:22-23).
 */
#ifndef MOE_B200_H
#define MOE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOE_B200_ABI_VERSION 1

typedef enum {
    MOE_OK = 0,
    MOE_SHAPE = 1,         /* moeforge::ShapeError         common.hpp:10-13 */
    MOE_CONFIG = 2,        /* moeforge::ConfigError        common.hpp:21-24 */
    MOE_NONFINITE = 3,     /* moeforge::NonFiniteError     common.hpp:15-19, tensor.cpp:23-29 */
    MOE_UNIFORM_SHAPE = 4, /* moeforge::UniformShapeError  common.hpp:31-35 */
    MOE_INVALID_ARG = 5,   /* std::invalid_argument (balance_loss routing.cpp:360-361) */
    MOE_CUDA = 6,          /* CUDA runtime/driver failure */
    MOE_NCCL = 7,          /* NCCL failure on the expert-parallel path */
    MOE_UNSUPPORTED = 8    /* valid for the reference, not implemented on this path */
} moe_status;

typedef enum { MOE_TRAIN = 0, MOE_EVAL = 1 } moe_phase;                       /* routing.hpp:13 */
typedef enum { MOE_PLAIN = 0, MOE_GROUPED = 1, MOE_RTS = 2 } moe_assignment;  /* routing.hpp:15 */
typedef enum { MOE_F32 = 0, MOE_BF16 = 1, MOE_F64 = 2 } moe_dtype;

#define MOE_KDROPPED (-1) /* routing.hpp:34 kDropped */

/* RouterConfig, routing.hpp:17-32 (same fields, same defaults via
 * moe_router_cfg_default). */
typedef struct {
    int num_experts;
    double capacity_factor_train;
    double capacity_factor_eval;
    double jitter_eps;
    double balance_coeff;
    int assignment_mode; /* moe_assignment */
    int group_count;     /* only used by MOE_GROUPED */
    int top_k;           /* 1 or 2 */
    uint64_t rng_seed;
} moe_router_cfg;

typedef struct {
    int64_t max_tokens; /* per rank; sizes the handle's workspace */
    int64_t d_model;
    int64_t d_ff;
    int dtype;          /* moe_dtype */
    int ep_size;        /* expert-parallel ranks (1 = single GPU) */
    int ep_rank;
} moe_layer_dims;

typedef struct moe_handle moe_handle;

/* Device flag bits latched by kernels, read by moe_check(). */
#define MOE_FLAG_NONFINITE 0x1u
#define MOE_FLAG_PROB_ROWS 0x2u /* balance_loss: probs rows must sum to 1 */
#define MOE_FLAG_CHOICE_RANGE 0x4u
#define MOE_FLAG_UNIFORM_SHAPE 0x8u /* expert parallelism: ranks passed different T */

void moe_router_cfg_default(moe_router_cfg* cfg);                    /* routing.hpp:17-27 */
moe_status moe_router_cfg_validate(const moe_router_cfg* cfg);       /* routing.cpp:13-23 */
/* capacity(tokens, cfg, phase), routing.cpp:43-49 (host only) */
moe_status moe_capacity(int64_t tokens, const moe_router_cfg* cfg, int phase, int* cap_out);
int moe_abi_version(void);

moe_status moe_create(const moe_router_cfg* cfg, const moe_layer_dims* dims, moe_handle** out);
moe_status moe_destroy(moe_handle* h);
const char* moe_last_error(const moe_handle* h);
moe_status moe_set_stream(moe_handle* h, void* cuda_stream);
/* Synchronise the handle's stream; MOE_NONFINITE / MOE_INVALID_ARG if a
 * kernel latched a flag since the last check (flags are then cleared). */
moe_status moe_check(moe_handle* h, uint32_t* flags_out);

/* ---- full layer: moe_layer_forward, routing.cpp:376-424 ---------------- */
/* Forward.  T <= max_tokens rows of x.  residual == NULL means "x" (the
 * reference default); pass a zero tensor for the contribution form
 * (model.cpp:342).  aux: 1 float (device).  Decision outputs are optional
 * (NULL to skip): expert_id, slot [T*top_k] int32 (slot = kDropped or the
 * capacity slot, exactly as RoutingDecision), gate_prob [T*top_k] fp32.
 * The forward context (decision, probabilities, hidden activations) is kept
 * in the handle for moe_backward. */
moe_status moe_forward(moe_handle* h, int64_t T, const void* x, const float* gate_w,
                       const void* w1, const float* b1, const void* w2, const float* b2,
                       int phase, uint64_t seed, const void* residual, void* y, float* aux,
                       int32_t* expert_id, int32_t* slot, float* gate_prob);

/* Backward of loss = <dy, y> + daux * aux for the last moe_forward on this
 * handle (the closures the reference tape runs, tensor.cpp:156-187).
 * Gradients are WRITTEN (not accumulated).  dgate_w is summed over ranks
 * under expert parallelism.  dresidual is required iff a residual was passed
 * to the forward (else ignored; its gradient then flows into dx). */
moe_status moe_backward(moe_handle* h, const void* dy, float daux, void* dx, float* dgate_w,
                        void* dw1, float* db1, void* dw2, float* db2, void* dresidual);

/* Which kernel family runs this handle's expert GEMMs.  bf16 layers use the
 * tcgen05/TMEM kernels when d_model and d_ff are multiples of 256, else the
 * fp32-accumulating SIMT kernels (logged to stderr at moe_create unless
 * MOE_B200_QUIET=1; MOE_B200_REQUIRE_TC=1 makes moe_create fail with
 * MOE_UNSUPPORTED instead).  fp32 layers always use SIMT (the parity path). */
typedef enum { MOE_GEMM_SIMT = 0, MOE_GEMM_TCGEN05 = 1 } moe_gemm_kind;
moe_status moe_gemm_path(const moe_handle* h, int* path_out);

/* ---- float64 path: the reference's own precision (dtype MOE_F64) --------
 * Every tensor is float64, including gate_w, biases, aux, gate_prob and all
 * gradients.  Forward reductions run in the reference's order with separately
 * rounded products and sums (its x86-64 build has no FMA), so logits, the
 * expert FFN, y and the decisions match routing.cpp / ops.cpp bit for bit up
 * to glibc-vs-CUDA exp (<= 1 ulp in the probabilities); the backward follows
 * the tape's closures to ~1e-15.  For f64 callers (the tape adapter,
 * gradient checks at h = 1e-5); single rank.  accumulate != 0 adds into the
 * gradient buffers (the tape's += semantics, tensor.cpp:31-36) instead of
 * writing them. */
moe_status moe_forward_f64(moe_handle* h, int64_t T, const double* x, const double* gate_w, const double* w1,
                           const double* b1, const double* w2, const double* b2, int phase, uint64_t seed,
                           const double* residual, double* y, double* aux, int32_t* expert_id, int32_t* slot,
                           double* gate_prob);
moe_status moe_backward_f64(moe_handle* h, const double* dy, double daux, double* dx, double* dgate_w,
                            double* dw1, double* db1, double* dw2, double* db2, double* dresidual,
                            int accumulate);

/* moe_backward with output options (flags, OR-ed):
 *   MOE_GRAD_ACCUMULATE   every gradient is ADDED into its buffer (the
 *                         reference tape's +=, tensor.cpp:31-36 — gradient
 *                         accumulation over micro-batches); dW1 / dW2 are
 *                         read-modify-written by the weight-gradient GEMM
 *                         epilogue itself, the others land in handle
 *                         scratch and are added after
 *   MOE_GRAD_WEIGHTS_F32  (bf16 layers) dw1 / dw2 are FLOAT32 buffers,
 *                         written straight from the fp32 TMEM accumulators
 *                         (mixed-precision callers with fp32 masters)
 * flags = 0 is moe_backward. */
#define MOE_GRAD_ACCUMULATE 0x1u
#define MOE_GRAD_WEIGHTS_F32 0x2u
moe_status moe_backward_ex(moe_handle* h, const void* dy, float daux, void* dx, float* dgate_w, void* dw1,
                           float* db1, void* dw2, float* db2, void* dresidual, unsigned flags);

/* Capacity and kept/dropped statistics of the last forward (host copy;
 * synchronises).  kept_per_expert may be NULL, else [E] int64. */
moe_status moe_last_decision_stats(moe_handle* h, int* capacity, int64_t* drop_count,
                                   int64_t* kept_per_expert);

/* Generate the jitter stream of a FUTURE train-phase moe_forward(seed) with
 * `tokens` rows ahead of use: the work is launched by the next moe_forward on
 * this handle (after its gate, on its own stream, as MOE_B200_PF_SMS = 10
 * CTAs — one chunk of the mt19937_64 stream per SM) and co-runs with that
 * call's forward and dgrad expert GEMMs, which leave those SMs free; the
 * matching later forward swaps the buffer in instead of generating on every
 * SM at its head.  Values are identical either way (the stream depends only on
 * the seed).  Training-loop pattern (per-step seeds are known ahead,
 * trainer.cpp:146-149): prefetch(seed_{i+1}); forward(seed_i); backward. */
moe_status moe_prefetch_jitter(moe_handle* h, uint64_t seed, int64_t tokens);

/* Utilization and drop statistics of the last forward, accumulated on the
 * device into caller-owned int64 arrays (stream-ordered, no sync):
 *   util_dev[E]  += first-choice counts per expert (count_utilization,
 *                   surgery.cpp:100-122, counts expert_id[t*top_k]);
 *   hist_dev[10] : [0..7] += dropped routes by token-position octile
 *                   min(7, 8t/T), [8] += dropped routes, [9] += T*top_k
 *                   routes (DropHistogram::accumulate, trainer.cpp:15-29). */
moe_status moe_accumulate_decision_stats(moe_handle* h, int64_t* util_dev, int64_t* hist_dev);

/* ---- expert optimizer step: AdamOptimizer::step, optim.cpp:21-57 ------- */
/* *acc_dev += sum of squares of grad[0..n) (f64, fixed-order reduction);
 * grad_dtype is moe_dtype.  Call once per tensor, in a fixed order, then
 * moe_clip_scale: *scale_dev = clip / sqrt(*sq_dev) if clip > 0 and the norm
 * exceeds it, else 1 (optim.cpp:26-37).  All stream-ordered on `stream`
 * (a cudaStream_t, NULL = legacy default stream). */
moe_status moe_grad_sqnorm(const void* grad, int64_t n, int grad_dtype, double* acc_dev, void* stream);
moe_status moe_clip_scale(const double* sq_dev, double clip_norm, double* scale_dev, void* stream);
/* One bias-corrected Adam update of one tensor (optim.cpp:38-55), `step` =
 * the optimizer's step count after increment (1 for the first update).
 * theta (fp32 master), m, v: fp32 [n], updated in place; grad: fp32 or bf16;
 * theta_bf16 (nullable): bf16 copy of the new theta for the next forward;
 * scale_dev (nullable): gradient scale from moe_clip_scale.  The update is
 * evaluated in f64. */
moe_status moe_adam_update(float* theta, float* m, float* v, const void* grad, int64_t n,
                           int grad_dtype, void* theta_bf16, const double* scale_dev, double lr,
                           double beta1, double beta2, double eps, int64_t step, void* stream);

/* ---- capacity check: the ZeRO-2 / EP memory planner ---------------------
 * ParallelPlan / MemoryEstimate / memory_per_gpu / max_model_size
 * (parallel.hpp:13-74, parallel.cpp:18-115), host arithmetic with the
 * reference's bytes-per-parameter model (2 param + 2 grad + 12 optimizer),
 * which is this build's training layout (bf16 params / grads, fp32 master +
 * Adam moments).  moe_workspace_bytes adds what a handle really allocated
 * (activations, buffers) so callers can check a plan against HBM. */
typedef struct {
    int world_size;      /* N */
    int expert_parallel; /* ep */
    int model_parallel;  /* mp; data_parallel = N / mp */
    int zero_stage;      /* 0 or 2 */
    int offload;         /* grads + optimizer states in host memory */
} moe_parallel_plan;
typedef struct {
    double nonexpert_params, expert_params, nonexpert_grads, expert_grads, nonexpert_optim,
        expert_optim;
    int grad_optim_on_cpu;
    double gpu_total, cpu_total, optimizer_grad_share;
} moe_memory_estimate;
moe_status moe_plan_validate(const moe_parallel_plan* plan);
const char* moe_plan_last_error(void); /* text of the last plan error (this thread) */
moe_status moe_memory_per_gpu(const moe_parallel_plan* plan, double nonexpert_params,
                              double expert_params, moe_memory_estimate* out);
moe_status moe_max_model_size(const moe_parallel_plan* plan, double gpu_budget_bytes, double base_params,
                              double params_per_expert, int64_t* max_experts, double* total_params);
/* Device bytes this handle allocated for its workspace and saved context. */
moe_status moe_workspace_bytes(const moe_handle* h, size_t* bytes_out);

/* ---- per-stage entry points (routing.hpp:60-118) ----------------------- */
/* gate_forward (routing.cpp:51-101): probs [T,E] fp32, choice [T*k] int32,
 * gate_prob [T*k] fp32.  x has the handle's dtype. */
moe_status moe_gate(moe_handle* h, int64_t T, const void* x, const float* gate_w, int phase,
                    uint64_t jitter_seed, float* probs, int32_t* choice, float* gate_prob);
/* make_assignment (routing.cpp:189-206) over device choices; slot [T*k];
 * *capacity_host receives RoutingDecision::capacity. */
moe_status moe_assign(moe_handle* h, int64_t T, const int32_t* choice, int phase,
                      uint64_t assign_seed, int32_t* slot, int* capacity_host);
/* assign_plain / assign_grouped / assign_rts with an explicit capacity
 * (routing.cpp:147-187). mode = moe_assignment. */
moe_status moe_assign_mode(moe_handle* h, int64_t T, const int32_t* choice, int cap, int mode,
                           int group_count, uint64_t rts_seed, int32_t* slot, int* capacity_host);
/* dispatch (routing.cpp:208-243): buf [E*capacity, d] (unoccupied rows are
 * exactly zero), occupancy [E*capacity] uint8 (may be NULL). */
moe_status moe_dispatch(moe_handle* h, int64_t T, const void* x, const int32_t* expert_id,
                        const int32_t* slot, int capacity, void* buf, uint8_t* occupancy);
/* combine (routing.cpp:258-298): weights [top_k, T] fp32. */
moe_status moe_combine(moe_handle* h, int64_t T, const void* expert_out, const int32_t* expert_id,
                       const int32_t* slot, int capacity, const void* residual,
                       const float* weights, void* y);
/* balance_loss (routing.cpp:348-374): loss [1] fp32 (device). */
moe_status moe_balance_loss(moe_handle* h, int64_t T, const float* probs,
                            const int32_t* expert_id, double alpha, float* loss);

/* ---- expert parallelism (parallel.hpp:100-111, made real) --------------- */
/* Size of the NCCL unique id blob (ncclUniqueId). */
size_t moe_ep_unique_id_size(void);
/* Rank 0 creates the id; all ranks then call moe_ep_init with the same blob
 * (distributed by the caller, e.g. torch.distributed broadcast). */
moe_status moe_ep_get_unique_id(void* id_out);
/* Binds the handle to an NCCL communicator of dims.ep_size ranks.  Rank r
 * owns experts [r*E/ep, (r+1)*E/ep) (parallel.cpp:260-265); its w1/b1/w2/b2
 * are those E/ep experts.  Each rank gates its own tokens; moe_forward's
 * seed is the rank's seed (derive_seed(seed, r), parallel.cpp:272). */
moe_status moe_ep_init(moe_handle* h, const void* unique_id);
/* NCCL-free bootstrap of the NVLink peer map (ranks on one node; ranks may
 * share a GPU, which NCCL refuses).  Each rank writes its blob
 * (moe_ep_blob_size() bytes: its layer dims and the CUDA-IPC handles of its
 * receive buffers) with moe_ep_export, the caller all-gathers the blobs in
 * rank order by any means (MPI, torch.distributed gloo, a file), every rank
 * passes the gathered array to moe_ep_import, and the caller then runs one
 * barrier before the first forward.  Exchanges are then NVLink / peer-memory
 * stores closed by the device flag barrier; dgate_w is summed over ranks from
 * peer-mapped staging.  Ranks that built different layers fail with
 * MOE_CONFIG; different max_tokens with MOE_UNIFORM_SHAPE.  Needs ep <= 8
 * and E/ep % 4 == 0 (else MOE_UNSUPPORTED: use moe_ep_init). */
size_t moe_ep_blob_size(void);
moe_status moe_ep_export(moe_handle* h, void* blob_out);
moe_status moe_ep_import(moe_handle* h, const void* all_blobs);
/* Per-forward shape contract (parallel.cpp:245-253): every rank must pass
 * the same T to moe_forward.  The dispatch exchange compares the ranks' T on
 * the device; a mismatch latches MOE_FLAG_UNIFORM_SHAPE (no expert rows are
 * computed) and the next moe_check returns MOE_UNIFORM_SHAPE. */
/* Fixed-shape A2A accounting of the last forward (A2ATrafficLog,
 * parallel.hpp:83-91): bytes [ep, ep] in the reference's f64 units, and the
 * bytes actually moved by this rank. */
moe_status moe_ep_traffic(moe_handle* h, double* logical_bytes_host, double* actual_bytes_sent);

/* ---- observability (per-call stage times) ------------------ */
/* Enable/disable the per-stage CUDA-event timeline of this handle (resets
 * the accumulators).  Events are recorded on the handle's stream between
 * stages, so they time exactly the kernels of each stage. */
moe_status moe_profile_enable(moe_handle* h, int on);
/* Accumulated stage times since enable: names [max_stages][32] (NUL
 * terminated), total milliseconds and number of calls per stage. */
moe_status moe_profile_read(moe_handle* h, int max_stages, char* names, double* ms_total,
                            int64_t* calls, int* n_out);
/* Number of kernels this library has launched in the process so far. */
uint64_t moe_kernel_launch_count(void);

/* ---- testing: route bf16 expert GEMMs through the SIMT kernels instead of
 * tcgen05 (A/B comparisons of the two kernel families). ------------------ */
void moe_debug_set_tensor_cores(int enabled);
/* testing: raw mt19937_64 outputs [c*J, c*J + n) of Rng(seed) reconstructed
 * on the host through the jump-ahead polynomial the device generator uses. */
moe_status moe_debug_mt64_chunk_host(uint64_t seed, int64_t J, int c, int64_t n, uint64_t* out);
/* testing: the first `count` raw outputs of Rng(seed) from the device
 * generator into device memory out_dev. */
moe_status moe_debug_mt64_device(uint64_t seed, int64_t count, uint64_t* out_dev);
/* debugging: %globaltimer phase stamps [ncta][8] of the last fused-gate launch
 * when MOE_B200_GATE_PROBE has bit 8 (start, after pdl_wait, accumulator
 * ready, epilogue before / after the cluster barrier, routing done). */
moe_status moe_debug_gate_stamps(uint64_t* host, int ncta, int* n_out);
/* testing: Rng(seed).permutation(n) (the RTS order, rng.cpp:94-102) built on
 * the device (rts.cu) into device memory perm_dev [n] uint32. */
moe_status moe_debug_rts_order(uint64_t seed, int64_t n, uint32_t* perm_dev);
/* testing: the first `count` jitter values (float)Rng(seed).uniform(1-eps,
 * 1+eps) (rng.cpp:41-43) from the device generator into device memory. */
moe_status moe_debug_jitter_device(uint64_t seed, int64_t count, double eps, float* out_dev);

/* testing: the tensor-core gate GEMMs (gate_tc.cu) on device buffers; x,
 * dX, dy, dx, dres are bf16.  logits_part is [splits][T][E]; dw_part is
 * [splits][d][E]. */
moe_status moe_debug_gate_tc_logits(const void* x, const float* noise, const float* gate_w,
                                    float* logits_part, int64_t T, int d, int E, int splits);
moe_status moe_debug_gate_tc_dw(const void* x, const float* noise, const float* dL, float* dw_part,
                                int64_t T, int d, int E, int splits);
moe_status moe_debug_gate_tc_dx(int64_t T, int d, int E, int K, int cap_pad, const float* dL,
                                const float* gate_w, const float* noise, const void* dX,
                                const int32_t* choice, const int32_t* pos, const void* dy,
                                int residual_is_x, void* dx, void* dres);

/* ---- RNG streams (rng.cpp:15-102), host, bit-exact -------------------- */
uint64_t moe_derive_seed_tag(uint64_t seed, const char* tag);
uint64_t moe_derive_seed_u64(uint64_t seed, uint64_t salt);
/* Rng(seed).permutation(n), rng.cpp:94-102 (prune_experts' random strategy,
 * surgery.cpp:167-172; the RTS order), host. */
moe_status moe_rng_permutation(uint64_t seed, int64_t n, uint32_t* out_host);

/* ---- checkpoint -> device layout (checkpoint.cpp f64 records) ---------- */
/* dst[i] = (dtype)src[i] for i < n, round-to-nearest-even; src and dst are
 * device buffers (the f64 checkpoint record staged on the device). */
moe_status moe_convert_f64(const double* src, int64_t n, int dtype, void* dst, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MOE_B200_H */
