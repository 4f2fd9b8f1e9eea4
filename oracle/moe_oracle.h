/*
 * moe_oracle.h — CPU restatement of the reference MoE-layer hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 kernels in paper_2109_10465_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path (libmoe_b200.so) never links, loads or calls it.
 *
 * It restates, in plain C99 with f64 arithmetic and the reference's
 * summation orders, the algorithm of
 *   /root/reference/proj/core/src/routing.cpp:13-424   (router, assign, dispatch, combine, loss, layer)
 *   /root/reference/proj/core/src/rng.cpp:15-102        (splitmix64 seeds, mt19937_64 draws, permutation)
 *   /root/reference/proj/core/src/ops.cpp:16-102,125-645 (kernels + the backward closures the tape runs)
 *   /root/reference/proj/core/src/parallel.cpp:231-366   (expert-parallel step)
 * Parity of this restatement is pinned two ways (tests/test_oracle.py):
 *   - the reference's own known-answer tests (test_routing.cpp, test_parallel.cpp);
 *   - golden vectors produced by the reference itself compiled from its
 *     sources (oracle/Makefile -> oracle/_ref/, tests/golden/make_golden.py).
 */
#ifndef MOE_ORACLE_H
#define MOE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: same numbering as include/moe_b200.h (moe_status). */
enum {
    ORC_OK = 0,
    ORC_SHAPE = 1,         /* ShapeError          common.hpp:10-13 */
    ORC_CONFIG = 2,        /* ConfigError         common.hpp:21-24 */
    ORC_NONFINITE = 3,     /* NonFiniteError      common.hpp:15-19 */
    ORC_UNIFORM_SHAPE = 4, /* UniformShapeError   common.hpp:31-35 */
    ORC_INVALID_ARG = 5    /* std::invalid_argument (balance_loss, uniform_int) */
};

enum { ORC_TRAIN = 0, ORC_EVAL = 1 };                    /* routing.hpp:13 */
enum { ORC_PLAIN = 0, ORC_GROUPED = 1, ORC_RTS = 2 };    /* routing.hpp:15 */

/* RouterConfig, routing.hpp:17-32 (rng_seed is unused by the layer). */
typedef struct {
    int num_experts;
    double capacity_factor_train;
    double capacity_factor_eval;
    double jitter_eps;
    double balance_coeff;
    int assignment_mode;
    int group_count;
    int top_k;
} orc_cfg;

void orc_cfg_default(orc_cfg* c);
int orc_cfg_validate(const orc_cfg* c);

/* ---- rng.cpp ---- */
uint64_t orc_splitmix64(uint64_t x);
uint64_t orc_derive_seed_tag(uint64_t seed, const char* tag);
uint64_t orc_derive_seed_u64(uint64_t seed, uint64_t salt);
/* Raw mt19937_64 outputs [skip, skip+n) of the stream seeded with seed. */
void orc_mt64_raw(uint64_t seed, int64_t skip, int64_t n, uint64_t* out);
/* n draws of Rng::uniform(lo, hi) */
void orc_uniform(uint64_t seed, double lo, double hi, int64_t n, double* out);
int orc_permutation(uint64_t seed, int64_t n, uint32_t* out);

/* ---- routing.cpp ---- */
int orc_capacity(int64_t tokens, const orc_cfg* cfg, int phase, int* cap);

/* gate_forward (routing.cpp:51-101).  probs [T,E]; choice [T*k];
 * gate_prob [T*k] (= probs[t, choice[t*k+kk]]); noise [T*d] optional
 * (filled with 1.0 when jitter is off). */
int orc_gate_forward(const double* x, const double* gate_w, int64_t T, int64_t d,
                     const orc_cfg* cfg, int phase, uint64_t jitter_seed,
                     double* probs, int32_t* choice, double* gate_prob, double* noise);

/* scan_assign in a given mode (routing.cpp:113-187).  slot [T*k]. */
int orc_assign(const int32_t* choice, int64_t T, int num_experts, int cap, int top_k,
               int mode, int group_count, uint64_t rts_seed, int32_t* slot, int* capacity_out);

/* make_assignment (routing.cpp:189-206) */
int orc_make_assignment(const int32_t* choice, int64_t T, const orc_cfg* cfg, int phase,
                        uint64_t rng_seed, int32_t* slot, int* capacity_out);

/* dispatch (routing.cpp:208-256): buf [E*cap, d] zero-filled, occupancy [E*cap] */
int orc_dispatch(const double* x, int64_t T, int64_t d, const int32_t* expert_id,
                 const int32_t* slot, int top_k, int num_experts, int cap,
                 double* buf, uint8_t* occupancy);

/* combine (routing.cpp:258-298); weights [k][T] */
int orc_combine(const double* expert_out, int64_t T, int64_t d, const int32_t* expert_id,
                const int32_t* slot, int top_k, int num_experts, int cap,
                const double* residual, const double* weights, double* y);

/* balance_loss (routing.cpp:348-374) */
int orc_balance_loss(const double* probs, int64_t T, int num_experts, const int32_t* expert_id,
                     int top_k, double alpha, double* loss);

/* moe_layer_forward (routing.cpp:376-424) followed, when dy != NULL, by the
 * backward the reference tape runs for loss = <dy, y> + daux * aux.
 * Weights are packed per expert in the reference orientation:
 *   w1 [E, d, f], b1 [E, f], w2 [E, f, d], b2 [E, d].
 * residual == NULL means "x" (the reference default).  Gradients are
 * written (not accumulated).  dresidual is only written when residual != NULL.
 * Decision outputs: expert_id/slot/gate_prob [T*k]; capacity_out. */
int orc_moe_layer(const double* x, const double* gate_w, const double* w1, const double* b1,
                  const double* w2, const double* b2, int64_t T, int64_t d, int64_t f,
                  const orc_cfg* cfg, int phase, uint64_t seed, const double* residual,
                  double* y, double* aux, int32_t* expert_id, int32_t* slot, double* gate_prob,
                  int* capacity_out,
                  const double* dy, double daux, double* dx, double* dgate_w, double* dw1,
                  double* db1, double* dw2, double* db2, double* dresidual);

/* simulate_expert_parallel_step (parallel.cpp:231-366), forward only.
 * xs [ep, T, d]; ys [ep, T, d]; expert_id/slot/gate_prob [ep, T];
 * traffic [ep, ep] bytes (fixed-shape f64 accounting). */
int orc_ep_forward(const double* xs, int ep, int64_t T, int64_t d, int64_t f,
                   const double* gate_w, const double* w1, const double* b1, const double* w2,
                   const double* b2, const orc_cfg* cfg, int phase, uint64_t seed,
                   double* ys, int32_t* expert_id, int32_t* slot, double* gate_prob,
                   int* capacity_out, double* traffic);

#ifdef __cplusplus
}
#endif
#endif
