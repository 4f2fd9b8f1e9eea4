/*
 * moe_oracle.c — CPU restatement of the reference MoE-layer hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see moe_oracle.h).  Plain C99, f64, the
 * reference's loop/summation orders.  Every function cites the reference
 * lines (relative to /root/reference/proj/) it restates.
 */
#include "moe_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* mt19937_64 (the std::mt19937_64 engine of rng.hpp:52), restated from */
/* the C++ standard's parameterisation [rand.predef].                  */
/* ------------------------------------------------------------------ */
#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

typedef struct {
    uint64_t x[MT_N];
    int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
    s->x[0] = seed;
    for (int i = 1; i < MT_N; ++i) {
        s->x[i] = 6364136223846793005ULL * (s->x[i - 1] ^ (s->x[i - 1] >> 62)) + (uint64_t)i;
    }
    s->idx = MT_N;
}

static void mt64_twist(mt64* s) {
    uint64_t* x = s->x;
    int i;
    for (i = 0; i < MT_N - MT_M; ++i) {
        uint64_t y = (x[i] & MT_UM) | (x[i + 1] & MT_LM);
        x[i] = x[i + MT_M] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
    }
    for (; i < MT_N - 1; ++i) {
        uint64_t y = (x[i] & MT_UM) | (x[i + 1] & MT_LM);
        x[i] = x[i + MT_M - MT_N] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
    }
    uint64_t y = (x[MT_N - 1] & MT_UM) | (x[0] & MT_LM);
    x[MT_N - 1] = x[MT_M - 1] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
    s->idx = 0;
}

static uint64_t mt64_next(mt64* s) {
    if (s->idx >= MT_N) mt64_twist(s);
    uint64_t z = s->x[s->idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

/* rng.cpp:15-20 */
uint64_t orc_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* rng.cpp:24-30 */
uint64_t orc_derive_seed_tag(uint64_t seed, const char* tag) {
    uint64_t h = orc_splitmix64(seed);
    for (const unsigned char* c = (const unsigned char*)tag; *c; ++c) h = orc_splitmix64(h ^ *c);
    return h;
}

/* rng.cpp:32-34 */
uint64_t orc_derive_seed_u64(uint64_t seed, uint64_t salt) {
    return orc_splitmix64(orc_splitmix64(seed) ^ salt);
}

void orc_mt64_raw(uint64_t seed, int64_t skip, int64_t n, uint64_t* out) {
    mt64 s;
    mt64_seed(&s, seed);
    for (int64_t i = 0; i < skip; ++i) (void)mt64_next(&s);
    for (int64_t i = 0; i < n; ++i) out[i] = mt64_next(&s);
}

/* rng.cpp:36-43 */
static double rng_uniform01(mt64* s) { return (double)(mt64_next(s) >> 11) * 0x1.0p-53; }
static double rng_uniform(mt64* s, double lo, double hi) { return lo + (hi - lo) * rng_uniform01(s); }

void orc_uniform(uint64_t seed, double lo, double hi, int64_t n, double* out) {
    mt64 s;
    mt64_seed(&s, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng_uniform(&s, lo, hi);
}

/* rng.cpp:45-56 */
static uint64_t rng_uniform_int(mt64* s, uint64_t n) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t x;
    do {
        x = mt64_next(s);
    } while (x >= limit);
    return x % n;
}

/* rng.cpp:94-102 */
int orc_permutation(uint64_t seed, int64_t n, uint32_t* out) {
    mt64 s;
    mt64_seed(&s, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = (uint32_t)i;
    for (int64_t i = n; i > 1; --i) {
        const int64_t j = (int64_t)rng_uniform_int(&s, (uint64_t)i);
        uint32_t t = out[i - 1];
        out[i - 1] = out[j];
        out[j] = t;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* routing.cpp                                                          */
/* ------------------------------------------------------------------ */
void orc_cfg_default(orc_cfg* c) { /* routing.hpp:17-27 */
    c->num_experts = 8;
    c->capacity_factor_train = 1.0;
    c->capacity_factor_eval = 2.0;
    c->jitter_eps = 0.01;
    c->balance_coeff = 0.01;
    c->assignment_mode = ORC_PLAIN;
    c->group_count = 1;
    c->top_k = 1;
}

/* routing.cpp:13-23 */
int orc_cfg_validate(const orc_cfg* c) {
    if (c->num_experts < 1) return ORC_CONFIG;
    if (c->capacity_factor_train <= 0.0 || c->capacity_factor_eval <= 0.0) return ORC_CONFIG;
    if (c->balance_coeff < 0.0) return ORC_CONFIG;
    if (c->jitter_eps < 0.0) return ORC_CONFIG;
    if (c->group_count < 1) return ORC_CONFIG;
    if (c->top_k != 1 && c->top_k != 2) return ORC_CONFIG;
    if (c->top_k > c->num_experts) return ORC_CONFIG;
    return ORC_OK;
}

/* routing.cpp:43-49 */
int orc_capacity(int64_t tokens, const orc_cfg* cfg, int phase, int* cap) {
    if (tokens < 1) return ORC_CONFIG;
    int st = orc_cfg_validate(cfg);
    if (st) return st;
    const double cf = phase == ORC_TRAIN ? cfg->capacity_factor_train : cfg->capacity_factor_eval;
    const double c = cf * (double)tokens / (double)cfg->num_experts;
    int v = (int)ceil(c);
    *cap = v < 1 ? 1 : v;
    return ORC_OK;
}

/* kernels::matmul_acc, ops.cpp:16-29 — c += a[m,k] @ b[k,n], i-p-j order */
static void matmul_acc(const double* a, const double* b, double* c, int64_t m, int64_t k,
                       int64_t n) {
    for (int64_t i = 0; i < m; ++i) {
        const double* arow = a + i * k;
        double* crow = c + i * n;
        for (int64_t p = 0; p < k; ++p) {
            const double av = arow[p];
            const double* brow = b + p * n;
            for (int64_t j = 0; j < n; ++j) crow[j] += av * brow[j];
        }
    }
}

/* kernels::matmul_bt_acc, ops.cpp:31-45 — c += a[m,k] @ b[n,k]^T */
static void matmul_bt_acc(const double* a, const double* b, double* c, int64_t m, int64_t k,
                          int64_t n) {
    for (int64_t i = 0; i < m; ++i) {
        const double* arow = a + i * k;
        double* crow = c + i * n;
        for (int64_t j = 0; j < n; ++j) {
            const double* brow = b + j * k;
            double acc = 0.0;
            for (int64_t p = 0; p < k; ++p) acc += arow[p] * brow[p];
            crow[j] += acc;
        }
    }
}

/* kernels::matmul_at_acc, ops.cpp:47-60 — c += a[m,k]^T @ b[m,n] */
static void matmul_at_acc(const double* a, const double* b, double* c, int64_t m, int64_t k,
                          int64_t n) {
    for (int64_t i = 0; i < m; ++i) {
        const double* arow = a + i * k;
        const double* brow = b + i * n;
        for (int64_t p = 0; p < k; ++p) {
            const double av = arow[p];
            double* crow = c + p * n;
            for (int64_t j = 0; j < n; ++j) crow[j] += av * brow[j];
        }
    }
}

/* kernels::softmax_row, ops.cpp:77-90 */
static void softmax_row(const double* x, double* y, int64_t n) {
    double mx = x[0];
    for (int64_t j = 1; j < n; ++j) mx = x[j] > mx ? x[j] : mx;
    double sum = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        y[j] = exp(x[j] - mx);
        sum += y[j];
    }
    for (int64_t j = 0; j < n; ++j) y[j] /= sum;
}

static int all_finite(const double* v, int64_t n) { /* tensor.cpp:23-29 */
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite(v[i])) return 0;
    return 1;
}

/* gate_forward, routing.cpp:51-101 */
int orc_gate_forward(const double* x, const double* gate_w, int64_t T, int64_t d,
                     const orc_cfg* cfg, int phase, uint64_t jitter_seed, double* probs,
                     int32_t* choice, double* gate_prob, double* noise) {
    int st = orc_cfg_validate(cfg);
    if (st) return st;
    const int64_t E = cfg->num_experts;
    const int K = cfg->top_k;
    double* gin = (double*)malloc(sizeof(double) * (size_t)(T * d > 0 ? T * d : 1));
    double* logits = (double*)calloc((size_t)(T * E > 0 ? T * E : 1), sizeof(double));
    if (phase == ORC_TRAIN && cfg->jitter_eps > 0.0) { /* routing.cpp:62-70 */
        mt64 s;
        mt64_seed(&s, jitter_seed);
        for (int64_t i = 0; i < T * d; ++i) {
            const double nv = rng_uniform(&s, 1.0 - cfg->jitter_eps, 1.0 + cfg->jitter_eps);
            if (noise) noise[i] = nv;
            gin[i] = x[i] * nv; /* mul, ops.cpp:213-220 */
        }
    } else {
        for (int64_t i = 0; i < T * d; ++i) {
            gin[i] = x[i];
            if (noise) noise[i] = 1.0;
        }
    }
    st = ORC_OK;
    if (!all_finite(gin, T * d)) st = ORC_NONFINITE;
    matmul_acc(gin, gate_w, logits, T, d, E); /* routing.cpp:71 */
    if (!st && !all_finite(logits, T * E)) st = ORC_NONFINITE;
    for (int64_t t = 0; t < T; ++t) softmax_row(logits + t * E, probs + t * E, E);
    if (!st && !all_finite(probs, T * E)) st = ORC_NONFINITE;
    for (int64_t t = 0; t < T; ++t) { /* routing.cpp:75-92 */
        const double* row = probs + t * E;
        int32_t best = 0;
        for (int64_t e = 1; e < E; ++e)
            if (row[e] > row[best]) best = (int32_t)e;
        choice[t * K] = best;
        if (K == 2) {
            int32_t second = best == 0 ? 1 : 0;
            for (int64_t e = 0; e < E; ++e) {
                if (e == best) continue;
                if (row[e] > row[second]) second = (int32_t)e;
            }
            choice[t * K + 1] = second;
        }
        for (int k = 0; k < K; ++k) gate_prob[t * K + k] = row[choice[t * K + k]];
    }
    free(gin);
    free(logits);
    return st;
}

/* check_choices, routing.cpp:105-111 */
static int check_choices(const int32_t* choice, int64_t n, int E) {
    for (int64_t i = 0; i < n; ++i)
        if (choice[i] < 0 || choice[i] >= E) return ORC_CONFIG;
    return ORC_OK;
}

/* scan_assign, routing.cpp:116-145: (token, k) pairs k-major in the
 * given token order; slot = base + used[e]++ while used[e] < span. */
static void scan_assign(const int32_t* choice, int E, int K, const uint32_t* order,
                        int64_t begin, int64_t end, int base, int span, int32_t* slot) {
    int* used = (int*)calloc((size_t)E, sizeof(int));
    for (int k = 0; k < K; ++k) {
        for (int64_t i = begin; i < end; ++i) {
            const int64_t t = order ? (int64_t)order[i] : i;
            const int64_t idx = t * K + k;
            const int32_t e = choice[idx];
            if (used[e] < span) {
                slot[idx] = base + used[e];
                ++used[e];
            }
        }
    }
    free(used);
}

/* assign_plain / assign_grouped / assign_rts, routing.cpp:147-187 */
int orc_assign(const int32_t* choice, int64_t T, int E, int cap, int K, int mode, int G,
               uint64_t rts_seed, int32_t* slot, int* capacity_out) {
    int st = check_choices(choice, T * K, E);
    if (st) return st;
    for (int64_t i = 0; i < T * K; ++i) slot[i] = -1;
    if (mode == ORC_PLAIN) {
        scan_assign(choice, E, K, NULL, 0, T, 0, cap, slot);
        *capacity_out = cap;
    } else if (mode == ORC_GROUPED) {
        if (G < 1 || T % G != 0) return ORC_CONFIG;
        const int gcap = (int)ceil((double)cap / (double)G);
        const int64_t glen = T / G;
        for (int g = 0; g < G; ++g)
            scan_assign(choice, E, K, NULL, g * glen, (g + 1) * glen, g * gcap, gcap, slot);
        *capacity_out = gcap * G;
    } else if (mode == ORC_RTS) {
        uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(T > 0 ? T : 1));
        orc_permutation(rts_seed, T, order);
        scan_assign(choice, E, K, order, 0, T, 0, cap, slot);
        free(order);
        *capacity_out = cap;
    } else {
        return ORC_CONFIG;
    }
    return ORC_OK;
}

/* make_assignment, routing.cpp:189-206 */
int orc_make_assignment(const int32_t* choice, int64_t T, const orc_cfg* cfg, int phase,
                        uint64_t rng_seed, int32_t* slot, int* capacity_out) {
    int cap;
    int st = orc_capacity(T, cfg, phase, &cap);
    if (st) return st;
    const int mode = phase == ORC_EVAL ? ORC_PLAIN : cfg->assignment_mode;
    return orc_assign(choice, T, cfg->num_experts, cap, cfg->top_k, mode, cfg->group_count,
                      rng_seed, slot, capacity_out);
}

/* dispatch, routing.cpp:208-243 */
int orc_dispatch(const double* x, int64_t T, int64_t d, const int32_t* expert_id,
                 const int32_t* slot, int K, int E, int cap, double* buf, uint8_t* occupancy) {
    const int64_t rows = (int64_t)E * cap;
    memset(buf, 0, sizeof(double) * (size_t)(rows * d));
    if (occupancy) memset(occupancy, 0, (size_t)rows);
    for (int64_t t = 0; t < T; ++t) {
        for (int k = 0; k < K; ++k) {
            const int64_t idx = t * K + k;
            if (slot[idx] == -1) continue;
            const int64_t row = (int64_t)expert_id[idx] * cap + slot[idx];
            if (row < 0 || row >= rows) return ORC_SHAPE;
            memcpy(buf + row * d, x + t * d, sizeof(double) * (size_t)d);
            if (occupancy) occupancy[row] = 1;
        }
    }
    return ORC_OK;
}

/* combine forward, routing.cpp:258-298 */
int orc_combine(const double* O, int64_t T, int64_t d, const int32_t* expert_id,
                const int32_t* slot, int K, int E, int cap, const double* residual,
                const double* weights, double* y) {
    (void)E;
    memset(y, 0, sizeof(double) * (size_t)(T * d));
    for (int64_t t = 0; t < T; ++t) {
        int any = 0;
        for (int k = 0; k < K; ++k) {
            const int64_t idx = t * K + k;
            if (slot[idx] == -1) continue;
            any = 1;
            const int64_t row = (int64_t)expert_id[idx] * cap + slot[idx];
            const double w = weights[(int64_t)k * T + t];
            for (int64_t j = 0; j < d; ++j) y[t * d + j] += w * O[row * d + j];
        }
        if (!any) memcpy(y + t * d, residual + t * d, sizeof(double) * (size_t)d);
    }
    return all_finite(y, T * d) ? ORC_OK : ORC_NONFINITE;
}

/* balance_loss, routing.cpp:348-374 (+ mean_cols ops.cpp:513-526,
 * dot_constant ops.cpp:541-550) */
int orc_balance_loss(const double* P, int64_t T, int E, const int32_t* expert_id, int K,
                     double alpha, double* loss) {
    for (int64_t t = 0; t < T; ++t) {
        double s = 0.0;
        for (int e = 0; e < E; ++e) s += P[t * E + e];
        if (fabs(s - 1.0) > 1e-9) return ORC_INVALID_ARG;
    }
    double* f = (double*)calloc((size_t)E, sizeof(double));
    double* mean = (double*)calloc((size_t)E, sizeof(double));
    for (int64_t t = 0; t < T; ++t) f[expert_id[t * K]] += 1.0;
    const double coeff = alpha * (double)E / (double)T;
    for (int e = 0; e < E; ++e) f[e] *= coeff;
    for (int64_t t = 0; t < T; ++t)
        for (int e = 0; e < E; ++e) mean[e] += P[t * E + e];
    for (int e = 0; e < E; ++e) mean[e] /= (double)T;
    double s = 0.0;
    for (int e = 0; e < E; ++e) s += mean[e] * f[e];
    *loss = s;
    free(f);
    free(mean);
    return ORC_OK;
}

/* moe_layer_forward, routing.cpp:376-424, plus the explicit backward of
 * the tape it builds (ops.cpp backward closures; routing.cpp:245-253,311-344). */
int orc_moe_layer(const double* x, const double* gate_w, const double* w1, const double* b1,
                  const double* w2, const double* b2, int64_t T, int64_t d, int64_t f,
                  const orc_cfg* cfg, int phase, uint64_t seed, const double* residual,
                  double* y, double* aux, int32_t* expert_id, int32_t* slot, double* gate_prob,
                  int* capacity_out, const double* dy, double daux, double* dx, double* dgate_w,
                  double* dw1, double* db1, double* dw2, double* db2, double* dresidual) {
    int st = orc_cfg_validate(cfg);
    if (st) return st;
    if (T < 1 || d < 1 || f < 1) return ORC_SHAPE;
    const int E = cfg->num_experts;
    const int K = cfg->top_k;
    const uint64_t jseed = orc_derive_seed_tag(seed, "jitter");
    const uint64_t aseed = orc_derive_seed_tag(seed, "assign");

    double* P = (double*)malloc(sizeof(double) * (size_t)(T * E));
    double* noise = (double*)malloc(sizeof(double) * (size_t)(T * d));
    int st_gate = orc_gate_forward(x, gate_w, T, d, cfg, phase, jseed, P, expert_id, gate_prob,
                                   noise);
    if (st_gate) {
        free(P);
        free(noise);
        return st_gate;
    }
    int cap;
    st = orc_make_assignment(expert_id, T, cfg, phase, aseed, slot, &cap);
    if (st) {
        free(P);
        free(noise);
        return st;
    }
    *capacity_out = cap;
    const int64_t R = (int64_t)E * cap;
    double* buf = (double*)malloc(sizeof(double) * (size_t)(R * d));
    orc_dispatch(x, T, d, expert_id, slot, K, E, cap, buf, NULL);

    /* per-expert FFN on all cap rows, routing.cpp:399-405 */
    double* Hpre = (double*)calloc((size_t)(R * f), sizeof(double));
    double* H = (double*)malloc(sizeof(double) * (size_t)(R * f));
    double* O = (double*)calloc((size_t)(R * d), sizeof(double));
    for (int e = 0; e < E; ++e) {
        const double* X = buf + (int64_t)e * cap * d;
        double* hp = Hpre + (int64_t)e * cap * f;
        double* h = H + (int64_t)e * cap * f;
        double* o = O + (int64_t)e * cap * d;
        matmul_acc(X, w1 + (int64_t)e * d * f, hp, cap, d, f);
        for (int64_t i = 0; i < cap; ++i)
            for (int64_t j = 0; j < f; ++j) hp[i * f + j] = hp[i * f + j] + b1[e * f + j];
        for (int64_t i = 0; i < cap * f; ++i) h[i] = hp[i] > 0.0 ? hp[i] : 0.0;
        matmul_acc(h, w2 + (int64_t)e * f * d, o, cap, f, d);
        for (int64_t i = 0; i < cap; ++i)
            for (int64_t j = 0; j < d; ++j) o[i * d + j] = o[i * d + j] + b2[e * d + j];
    }
    if (!all_finite(Hpre, R * f) || !all_finite(O, R * d)) st = ORC_NONFINITE;

    /* combine weights, routing.cpp:408-417 */
    double* W = (double*)malloc(sizeof(double) * (size_t)(K * T));
    double* S = (double*)malloc(sizeof(double) * (size_t)T);
    for (int64_t t = 0; t < T; ++t) {
        if (K == 1) {
            W[t] = gate_prob[t] * (double)E;
        } else {
            S[t] = gate_prob[t * 2] + gate_prob[t * 2 + 1];
            W[t] = gate_prob[t * 2] / S[t];
            W[T + t] = gate_prob[t * 2 + 1] / S[t];
        }
    }
    if (!st) st = orc_balance_loss(P, T, E, expert_id, K, cfg->balance_coeff, aux);
    const double* res = residual ? residual : x;
    if (!st) st = orc_combine(O, T, d, expert_id, slot, K, E, cap, res, W, y);

    if (!st && dy) {
        /* combine backward, routing.cpp:311-344 */
        double* dO = (double*)calloc((size_t)(R * d), sizeof(double));
        double* dW = (double*)calloc((size_t)(K * T), sizeof(double));
        double* dres = (double*)calloc((size_t)(T * d), sizeof(double));
        for (int64_t t = 0; t < T; ++t) {
            int any = 0;
            for (int k = 0; k < K; ++k) {
                const int64_t idx = t * K + k;
                if (slot[idx] == -1) continue;
                any = 1;
                const int64_t row = (int64_t)expert_id[idx] * cap + slot[idx];
                const double w = W[(int64_t)k * T + t];
                for (int64_t j = 0; j < d; ++j) dO[row * d + j] += w * dy[t * d + j];
                double dot = 0.0;
                for (int64_t j = 0; j < d; ++j) dot += dy[t * d + j] * O[row * d + j];
                dW[(int64_t)k * T + t] += dot;
            }
            if (!any)
                for (int64_t j = 0; j < d; ++j) dres[t * d + j] += dy[t * d + j];
        }
        /* expert backward: add_bias (ops.cpp:199-209), matmul (ops.cpp:135-144),
         * relu (ops.cpp:307-315) */
        double* dbuf = (double*)calloc((size_t)(R * d), sizeof(double));
        double* dH = (double*)malloc(sizeof(double) * (size_t)(cap * f));
        memset(dw1, 0, sizeof(double) * (size_t)(E * d * f));
        memset(dw2, 0, sizeof(double) * (size_t)(E * f * d));
        memset(db1, 0, sizeof(double) * (size_t)(E * f));
        memset(db2, 0, sizeof(double) * (size_t)(E * d));
        for (int e = 0; e < E; ++e) {
            const double* dOe = dO + (int64_t)e * cap * d;
            const double* He = H + (int64_t)e * cap * f;
            const double* Hp = Hpre + (int64_t)e * cap * f;
            const double* Xe = buf + (int64_t)e * cap * d;
            for (int64_t i = 0; i < cap; ++i)
                for (int64_t j = 0; j < d; ++j) db2[e * d + j] += dOe[i * d + j];
            memset(dH, 0, sizeof(double) * (size_t)(cap * f));
            matmul_bt_acc(dOe, w2 + (int64_t)e * f * d, dH, cap, d, f);
            matmul_at_acc(He, dOe, dw2 + (int64_t)e * f * d, cap, f, d);
            for (int64_t i = 0; i < cap * f; ++i)
                if (!(Hp[i] > 0.0)) dH[i] = 0.0;
            for (int64_t i = 0; i < cap; ++i)
                for (int64_t j = 0; j < f; ++j) db1[e * f + j] += dH[i * f + j];
            matmul_bt_acc(dH, w1 + (int64_t)e * d * f, dbuf + (int64_t)e * cap * d, cap, f, d);
            matmul_at_acc(Xe, dH, dw1 + (int64_t)e * d * f, cap, d, f);
        }
        /* dispatch backward, routing.cpp:245-253 */
        memset(dx, 0, sizeof(double) * (size_t)(T * d));
        for (int64_t t = 0; t < T; ++t)
            for (int k = 0; k < K; ++k) {
                const int64_t idx = t * K + k;
                if (slot[idx] == -1) continue;
                const int64_t row = (int64_t)expert_id[idx] * cap + slot[idx];
                for (int64_t j = 0; j < d; ++j) dx[t * d + j] += dbuf[row * d + j];
            }
        /* combine-weight backward: scale (ops.cpp:276-281) or add/div_elem
         * (ops.cpp:179-184, 250-262); then pick_per_row (ops.cpp:579-585) */
        double* dP = (double*)calloc((size_t)(T * E), sizeof(double));
        for (int64_t t = 0; t < T; ++t) {
            if (K == 1) {
                dP[t * E + expert_id[t]] += (double)E * dW[t];
            } else {
                const double p0 = gate_prob[t * 2], p1 = gate_prob[t * 2 + 1];
                const double s = S[t];
                double dp0 = dW[t] / s, dp1 = dW[T + t] / s;
                const double ds = -dW[t] * p0 / (s * s) - dW[T + t] * p1 / (s * s);
                dp0 += ds;
                dp1 += ds;
                dP[t * E + expert_id[t * 2]] += dp0;
                dP[t * E + expert_id[t * 2 + 1]] += dp1;
            }
        }
        /* balance loss backward: dot_constant (ops.cpp:552-558), mean_cols
         * (ops.cpp:528-537) with f constant (routing.cpp:364-373) */
        {
            double* fe = (double*)calloc((size_t)E, sizeof(double));
            for (int64_t t = 0; t < T; ++t) fe[expert_id[t * K]] += 1.0;
            const double coeff = cfg->balance_coeff * (double)E / (double)T;
            const double inv = 1.0 / (double)T;
            for (int e = 0; e < E; ++e) fe[e] *= coeff;
            for (int64_t t = 0; t < T; ++t)
                for (int e = 0; e < E; ++e) dP[t * E + e] += daux * fe[e] * inv;
            free(fe);
        }
        /* softmax backward, ops.cpp:329-343 */
        double* dL = (double*)malloc(sizeof(double) * (size_t)(T * E));
        for (int64_t t = 0; t < T; ++t) {
            double dot = 0.0;
            for (int e = 0; e < E; ++e) dot += dP[t * E + e] * P[t * E + e];
            for (int e = 0; e < E; ++e) dL[t * E + e] = P[t * E + e] * (dP[t * E + e] - dot);
        }
        /* gate matmul backward + jitter mul backward (ops.cpp:135-144, 223-228) */
        double* dg = (double*)calloc((size_t)(T * d), sizeof(double));
        matmul_bt_acc(dL, gate_w, dg, T, E, d);
        memset(dgate_w, 0, sizeof(double) * (size_t)(d * E));
        {
            double* gin = (double*)malloc(sizeof(double) * (size_t)(T * d));
            for (int64_t i = 0; i < T * d; ++i) gin[i] = x[i] * noise[i];
            if (!(phase == ORC_TRAIN && cfg->jitter_eps > 0.0))
                for (int64_t i = 0; i < T * d; ++i) gin[i] = x[i];
            matmul_at_acc(gin, dL, dgate_w, T, d, E);
            free(gin);
        }
        for (int64_t i = 0; i < T * d; ++i) dx[i] += dg[i] * noise[i];
        if (residual) {
            if (dresidual) memcpy(dresidual, dres, sizeof(double) * (size_t)(T * d));
        } else {
            for (int64_t i = 0; i < T * d; ++i) dx[i] += dres[i];
        }
        free(dO);
        free(dW);
        free(dres);
        free(dbuf);
        free(dH);
        free(dP);
        free(dL);
        free(dg);
    }
    free(P);
    free(noise);
    free(buf);
    free(Hpre);
    free(H);
    free(O);
    free(W);
    free(S);
    return st;
}

/* kernels::expert_ffn_rows, ops.cpp:92-102 */
static void expert_ffn_rows(const double* x, const double* w1, const double* b1,
                            const double* w2, const double* b2, double* hidden, double* y,
                            int64_t rows, int64_t d, int64_t f) {
    memset(hidden, 0, sizeof(double) * (size_t)(rows * f));
    matmul_acc(x, w1, hidden, rows, d, f);
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < f; ++j) hidden[i * f + j] = hidden[i * f + j] + b1[j];
    for (int64_t i = 0; i < rows * f; ++i) hidden[i] = hidden[i] > 0.0 ? hidden[i] : 0.0;
    memset(y, 0, sizeof(double) * (size_t)(rows * d));
    matmul_acc(hidden, w2, y, rows, f, d);
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < d; ++j) y[i * d + j] = y[i * d + j] + b2[j];
}

/* simulate_expert_parallel_step, parallel.cpp:231-366 */
int orc_ep_forward(const double* xs, int ep, int64_t T, int64_t d, int64_t f,
                   const double* gate_w, const double* w1, const double* b1, const double* w2,
                   const double* b2, const orc_cfg* cfg, int phase, uint64_t seed, double* ys,
                   int32_t* expert_id, int32_t* slot, double* gate_prob, int* capacity_out,
                   double* traffic) {
    int st = orc_cfg_validate(cfg);
    if (st) return st;
    if (ep < 1) return ORC_CONFIG;
    const int E = cfg->num_experts;
    if (E % ep != 0) return ORC_CONFIG;
    if (cfg->top_k != 1) return ORC_CONFIG;
    const int El = E / ep;
    double* P = (double*)malloc(sizeof(double) * (size_t)(T * E));
    int cap = 0;
    /* per-rank gate + assignment + dispatch, parallel.cpp:267-285 */
    double** bufs = (double**)calloc((size_t)ep, sizeof(double*));
    for (int r = 0; r < ep && !st; ++r) {
        const uint64_t rs = orc_derive_seed_u64(seed, (uint64_t)r);
        st = orc_gate_forward(xs + (int64_t)r * T * d, gate_w, T, d, cfg, phase,
                              orc_derive_seed_tag(rs, "jitter"), P, expert_id + r * T, gate_prob + r * T,
                              NULL);
        if (st) break;
        st = orc_make_assignment(expert_id + r * T, T, cfg, phase, orc_derive_seed_tag(rs, "assign"),
                                 slot + r * T, &cap);
        if (st) break;
        bufs[r] = (double*)malloc(sizeof(double) * (size_t)((int64_t)E * cap * d));
        orc_dispatch(xs + (int64_t)r * T * d, T, d, expert_id + r * T, slot + r * T, 1, E, cap,
                     bufs[r], NULL);
    }
    if (!st) {
        *capacity_out = cap;
        for (int i = 0; i < ep * ep; ++i) traffic[i] = 0.0;
        const int64_t slice = (int64_t)El * cap * d;
        /* fixed-shape forward exchange + local FFN + reverse exchange,
         * parallel.cpp:287-338 */
        double* outb = (double*)calloc((size_t)((int64_t)ep * E * cap * d), sizeof(double));
        double* hidden = (double*)malloc(sizeof(double) * (size_t)(cap * f));
        double* rows_out = (double*)malloc(sizeof(double) * (size_t)(cap * d));
        for (int s = 0; s < ep; ++s)
            for (int r = 0; r < ep; ++r)
                if (r != s) traffic[r * ep + s] += (double)slice * sizeof(double);
        for (int s = 0; s < ep; ++s)
            for (int r = 0; r < ep; ++r)
                for (int le = 0; le < El; ++le) {
                    const int e = s * El + le;
                    const double* xr = bufs[r] + (int64_t)e * cap * d;
                    expert_ffn_rows(xr, w1 + (int64_t)e * d * f, b1 + (int64_t)e * f,
                                    w2 + (int64_t)e * f * d, b2 + (int64_t)e * d, hidden, rows_out,
                                    cap, d, f);
                    memcpy(outb + ((int64_t)r * E + e) * cap * d, rows_out,
                           sizeof(double) * (size_t)(cap * d));
                    if (r != s) traffic[s * ep + r] += (double)cap * d * sizeof(double);
                }
        /* combine, parallel.cpp:340-362 */
        for (int r = 0; r < ep; ++r) {
            const double* x = xs + (int64_t)r * T * d;
            double* y = ys + (int64_t)r * T * d;
            memset(y, 0, sizeof(double) * (size_t)(T * d));
            for (int64_t t = 0; t < T; ++t) {
                if (slot[r * T + t] == -1) {
                    memcpy(y + t * d, x + t * d, sizeof(double) * (size_t)d);
                    continue;
                }
                const int64_t row = (int64_t)expert_id[r * T + t] * cap + slot[r * T + t];
                const double w = gate_prob[r * T + t] * (double)E;
                const double* orow = outb + ((int64_t)r * E * cap + row) * d;
                for (int64_t j = 0; j < d; ++j) y[t * d + j] += w * orow[j];
            }
        }
        free(outb);
        free(hidden);
        free(rows_out);
    }
    for (int r = 0; r < ep; ++r) free(bufs[r]);
    free(bufs);
    free(P);
    return st;
}
