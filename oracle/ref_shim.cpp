// ref_shim.cpp — extern "C" face over the reference itself.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference's own hot-path sources, unmodified, where they lie under
// /root/reference/proj/core/src (rng, tensor, ops, init, routing, parallel),
// into oracle/_ref/libmoeforge_ref.so.  Used to (a) pin the C restatement
// (moe_oracle.c) with golden vectors and (b) time the reference's CPU path
// for bench.py --impl reference.  Signatures mirror moe_oracle.h.
#include <moeforge/checkpoint.hpp>
#include <moeforge/common.hpp>
#include <moeforge/model.hpp>
#include <moeforge/surgery.hpp>
#include <moeforge/ops.hpp>
#include <moeforge/optim.hpp>
#include <moeforge/parallel.hpp>
#include <moeforge/rng.hpp>
#include <moeforge/routing.hpp>

#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

using namespace moeforge;

namespace {

struct ref_cfg {  // same layout as orc_cfg
    int num_experts;
    double capacity_factor_train;
    double capacity_factor_eval;
    double jitter_eps;
    double balance_coeff;
    int assignment_mode;
    int group_count;
    int top_k;
};

RouterConfig to_cfg(const ref_cfg* c) {
    RouterConfig r;
    r.num_experts = c->num_experts;
    r.capacity_factor_train = c->capacity_factor_train;
    r.capacity_factor_eval = c->capacity_factor_eval;
    r.jitter_eps = c->jitter_eps;
    r.balance_coeff = c->balance_coeff;
    r.assignment_mode = static_cast<AssignmentMode>(c->assignment_mode);
    r.group_count = c->group_count;
    r.top_k = c->top_k;
    return r;
}

Phase to_phase(int p) { return p == 0 ? Phase::kTrain : Phase::kEval; }

template <class F>
int guarded(F&& fn) {
    try {
        fn();
        return 0;
    } catch (const UniformShapeError&) {
        return 4;
    } catch (const NonFiniteError&) {
        return 3;
    } catch (const ConfigError&) {
        return 2;
    } catch (const ShapeError&) {
        return 1;
    } catch (const std::invalid_argument&) {
        return 5;
    } catch (...) {
        return 99;
    }
}

Tensor leaf(std::vector<std::int64_t> shape, const double* p, bool rg) {
    const std::int64_t n = shape_numel(shape);
    return Tensor::leaf(std::move(shape), std::vector<double>(p, p + n), rg);
}

MoeLayerParams make_params(const double* gate_w, const double* w1, const double* b1,
                           const double* w2, const double* b2, std::int64_t d, std::int64_t f,
                           int E, bool rg) {
    MoeLayerParams params;
    params.gate_w = leaf({d, E}, gate_w, rg);
    for (int e = 0; e < E; ++e) {
        params.experts.push_back({leaf({d, f}, w1 + static_cast<std::int64_t>(e) * d * f, rg),
                                  leaf({f}, b1 + static_cast<std::int64_t>(e) * f, rg),
                                  leaf({f, d}, w2 + static_cast<std::int64_t>(e) * f * d, rg),
                                  leaf({d}, b2 + static_cast<std::int64_t>(e) * d, rg)});
    }
    return params;
}

void copy_grad(const Tensor& t, double* out) {
    if (!out) return;
    if (t.has_grad()) {
        std::memcpy(out, t.grad().data(), sizeof(double) * t.grad().size());
    } else {
        std::memset(out, 0, sizeof(double) * static_cast<std::size_t>(t.numel()));
    }
}

}  // namespace

extern "C" {

uint64_t ref_derive_seed_tag(uint64_t seed, const char* tag) { return Rng::derive_seed(seed, tag); }
uint64_t ref_derive_seed_u64(uint64_t seed, uint64_t salt) { return Rng::derive_seed(seed, salt); }

void ref_mt64_raw(uint64_t seed, int64_t skip, int64_t n, uint64_t* out) {
    Rng rng(seed);
    for (int64_t i = 0; i < skip; ++i) (void)rng.next_u64();
    for (int64_t i = 0; i < n; ++i) out[i] = rng.next_u64();
}

int ref_permutation(uint64_t seed, int64_t n, uint32_t* out) {
    Rng rng(seed);
    auto p = rng.permutation(static_cast<std::size_t>(n));
    std::memcpy(out, p.data(), sizeof(uint32_t) * p.size());
    return 0;
}

int ref_capacity(int64_t tokens, const ref_cfg* c, int phase, int* cap) {
    return guarded([&] { *cap = capacity(tokens, to_cfg(c), to_phase(phase)); });
}

int ref_gate_forward(const double* x, const double* gate_w, int64_t T, int64_t d,
                     const ref_cfg* c, int phase, uint64_t jitter_seed, double* probs,
                     int32_t* choice, double* gate_prob) {
    return guarded([&] {
        RouterConfig cfg = to_cfg(c);
        GateResult g = gate_forward(leaf({T, d}, x, false), leaf({d, cfg.num_experts}, gate_w, false),
                                    cfg, to_phase(phase), jitter_seed);
        std::memcpy(probs, g.probs.data().data(), sizeof(double) * g.probs.data().size());
        std::memcpy(choice, g.choice.data(), sizeof(int32_t) * g.choice.size());
        for (int64_t t = 0; t < T; ++t)
            for (int k = 0; k < cfg.top_k; ++k)
                gate_prob[t * cfg.top_k + k] = g.gate_prob[static_cast<std::size_t>(k)].data()[t];
    });
}

int ref_assign(const int32_t* choice, int64_t T, int E, int cap, int K, int mode, int G,
               uint64_t rts_seed, int32_t* slot, int* cap_out) {
    return guarded([&] {
        std::span<const std::int32_t> ch(choice, static_cast<std::size_t>(T * K));
        RoutingDecision d;
        if (mode == 0) d = assign_plain(ch, E, cap, K);
        else if (mode == 1) d = assign_grouped(ch, E, cap, G, K);
        else d = assign_rts(ch, E, cap, rts_seed, K);
        std::memcpy(slot, d.slot.data(), sizeof(int32_t) * d.slot.size());
        *cap_out = d.capacity;
    });
}

int ref_moe_layer(const double* x, const double* gate_w, const double* w1, const double* b1,
                  const double* w2, const double* b2, int64_t T, int64_t d, int64_t f,
                  const ref_cfg* c, int phase, uint64_t seed, const double* residual, double* y,
                  double* aux, int32_t* expert_id, int32_t* slot, double* gate_prob,
                  int* capacity_out, const double* dy, double daux, double* dx, double* dgate_w,
                  double* dw1, double* db1, double* dw2, double* db2, double* dresidual) {
    return guarded([&] {
        RouterConfig cfg = to_cfg(c);
        const int E = cfg.num_experts;
        const bool rg = dy != nullptr;
        Tensor xt = leaf({T, d}, x, rg);
        MoeLayerParams params = make_params(gate_w, w1, b1, w2, b2, d, f, E, rg);
        Tensor rt;
        if (residual) rt = leaf({T, d}, residual, rg);
        MoeLayerResult r = moe_layer_forward(xt, params, cfg, to_phase(phase), seed,
                                             residual ? &rt : nullptr);
        std::memcpy(y, r.y.data().data(), sizeof(double) * r.y.data().size());
        *aux = r.aux_loss.scalar_value();
        std::memcpy(expert_id, r.decision.expert_id.data(), sizeof(int32_t) * r.decision.expert_id.size());
        std::memcpy(slot, r.decision.slot.data(), sizeof(int32_t) * r.decision.slot.size());
        std::memcpy(gate_prob, r.decision.gate_prob.data(), sizeof(double) * r.decision.gate_prob.size());
        *capacity_out = r.decision.capacity;
        if (!dy) return;
        // loss = <dy, y> + daux * aux (dot_constant / scale / add are tape ops).
        Tensor loss = add(dot_constant(r.y, std::span<const double>(dy, static_cast<std::size_t>(T * d))),
                          scale(r.aux_loss, daux));
        loss.backward();
        copy_grad(xt, dx);
        copy_grad(params.gate_w, dgate_w);
        for (int e = 0; e < E; ++e) {
            const auto& ex = params.experts[static_cast<std::size_t>(e)];
            copy_grad(ex.w1, dw1 + static_cast<std::int64_t>(e) * d * f);
            copy_grad(ex.b1, db1 + static_cast<std::int64_t>(e) * f);
            copy_grad(ex.w2, dw2 + static_cast<std::int64_t>(e) * f * d);
            copy_grad(ex.b2, db2 + static_cast<std::int64_t>(e) * d);
        }
        if (residual) copy_grad(rt, dresidual);
    });
}

int ref_ep_forward(const double* xs, int ep, int64_t T, int64_t d, int64_t f, const double* gate_w,
                   const double* w1, const double* b1, const double* w2, const double* b2,
                   const ref_cfg* c, int phase, uint64_t seed, double* ys, int32_t* expert_id,
                   int32_t* slot, double* gate_prob, int* capacity_out, double* traffic) {
    return guarded([&] {
        RouterConfig cfg = to_cfg(c);
        MoeLayerParams params = make_params(gate_w, w1, b1, w2, b2, d, f, cfg.num_experts, false);
        std::vector<Tensor> xt;
        for (int r = 0; r < ep; ++r) xt.push_back(leaf({T, d}, xs + static_cast<std::int64_t>(r) * T * d, false));
        SimResult s = simulate_expert_parallel_step(xt, params, cfg, to_phase(phase), seed, ep);
        for (int r = 0; r < ep; ++r) {
            std::memcpy(ys + static_cast<std::int64_t>(r) * T * d, s.outputs[r].data().data(),
                        sizeof(double) * static_cast<std::size_t>(T * d));
            std::memcpy(expert_id + r * T, s.decisions[r].expert_id.data(), sizeof(int32_t) * T);
            std::memcpy(slot + r * T, s.decisions[r].slot.data(), sizeof(int32_t) * T);
            std::memcpy(gate_prob + r * T, s.decisions[r].gate_prob.data(), sizeof(double) * T);
        }
        *capacity_out = s.decisions[0].capacity;
        std::memcpy(traffic, s.traffic.bytes.data(), sizeof(double) * s.traffic.bytes.size());
    });
}

// CPU baseline timing (bench.py --impl reference): `threads` independent
// replicas each run moe_layer_forward + backward of <dy,y>+aux on their own
// copy of the inputs (one replica per host thread; the reference itself is
// single-threaded).  Returns wall seconds of the slowest.
double ref_time_layer_mt(const double* x, const double* gate_w, const double* w1, const double* b1,
                         const double* w2, const double* b2, int64_t T, int64_t d, int64_t f,
                         const ref_cfg* c, int phase, uint64_t seed, const double* dy, int threads,
                         int* status) {
    std::vector<int> st(static_cast<std::size_t>(threads), 0);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int i = 0; i < threads; ++i) {
        pool.emplace_back([&, i] {
            st[static_cast<std::size_t>(i)] = guarded([&] {
                RouterConfig cfg = to_cfg(c);
                Tensor xt = leaf({T, d}, x, true);
                MoeLayerParams params = make_params(gate_w, w1, b1, w2, b2, d, f, cfg.num_experts, true);
                MoeLayerResult r = moe_layer_forward(xt, params, cfg, to_phase(phase),
                                                     Rng::derive_seed(seed, static_cast<std::uint64_t>(i)));
                Tensor loss = add(dot_constant(r.y, std::span<const double>(dy, static_cast<std::size_t>(T * d))),
                                  r.aux_loss);
                loss.backward();
            });
        });
    }
    for (auto& t : pool) t.join();
    auto t1 = std::chrono::steady_clock::now();
    *status = 0;
    for (int s : st)
        if (s) *status = s;
    return std::chrono::duration<double>(t1 - t0).count();
}


// AdamOptimizer (optim.cpp:10-57) on n flat leaves for `steps` steps; the
// gradient of step s is grads[s] (concatenated), injected through
// loss = sum_i dot_constant(theta_i, g_i) so backward() yields exactly g.
// theta is updated in place; final moments are returned concatenated.
int ref_adam(int n, const int64_t* numel, double* theta, const double* grads, int steps,
             const double* lrs, double clip, double beta1, double beta2, double eps,
             double* m_out, double* v_out) {
    return guarded([&] {
        std::vector<Tensor> params;
        int64_t total = 0;
        for (int i = 0; i < n; ++i) {
            params.push_back(Tensor::leaf({numel[i]}, std::vector<double>(theta + total, theta + total + numel[i]), true));
            total += numel[i];
        }
        AdamOptimizer opt(params, beta1, beta2, eps);
        for (int s = 0; s < steps; ++s) {
            opt.zero_grad();
            Tensor loss = Tensor::scalar(0.0);
            int64_t off = 0;
            for (int i = 0; i < n; ++i) {
                const double* g = grads + static_cast<int64_t>(s) * total + off;
                loss = add(loss, dot_constant(params[i], std::span<const double>(g, static_cast<size_t>(numel[i]))));
                off += numel[i];
            }
            loss.backward();
            opt.step(lrs[s], clip);
        }
        int64_t off = 0;
        for (int i = 0; i < n; ++i) {
            auto d = params[i].leaf_data();
            std::memcpy(theta + off, d.data(), sizeof(double) * d.size());
            const auto& st = opt.state(static_cast<size_t>(i));
            if (m_out) std::memcpy(m_out + off, st.m.data(), sizeof(double) * st.m.size());
            if (v_out) std::memcpy(v_out + off, st.v.data(), sizeof(double) * st.v.size());
            off += numel[i];
        }
    });
}

// Checkpoint -> device layout pinning: a small
// reference model built and saved by the reference itself, and its
// prune_experts (surgery.cpp:135-212).
int ref_save_toy_checkpoint(const char* dir, int64_t vocab, int64_t d_model, int64_t ffn_dim,
                            int enc_layers, int dec_layers, int heads, int num_experts,
                            int moe_every, uint64_t seed) {
    return guarded([&] {
        ArchConfig a = ArchConfig::toy(vocab, num_experts);
        a.d_model = d_model;
        a.ffn_dim = ffn_dim;
        a.enc_layers = enc_layers;
        a.dec_layers = dec_layers;
        a.heads = heads;
        a.moe_every = moe_every;
        save_checkpoint(build_model(a, seed), dir);
    });
}

// strategy 0 = top utilization (counts [num_moe_layers][E]), 1 = random(seed)
int ref_prune_checkpoint(const char* dir_in, const char* dir_out, int k, int strategy,
                         const int64_t* counts, uint64_t seed) {
    return guarded([&] {
        Checkpoint c = load_checkpoint(dir_in);
        UtilizationCounts u;
        const int L = c.arch.num_moe_layers(), E = c.arch.num_experts;
        if (counts) {
            u.per_layer.assign(static_cast<size_t>(L), std::vector<int64_t>(static_cast<size_t>(E)));
            for (int l = 0; l < L; ++l)
                for (int e = 0; e < E; ++e) u.per_layer[l][e] = counts[l * E + e];
        }
        Checkpoint p = prune_experts(c, k, strategy == 0 ? PruneStrategy::kTopUtilization : PruneStrategy::kRandom,
                                     counts ? &u : nullptr, seed);
        save_checkpoint(p, dir_out);
    });
}

// ---- parallel.cpp:18-115: the ZeRO-2 / EP memory planner -----------------
struct ref_plan {
    int world_size, expert_parallel, model_parallel, zero_stage, offload;
};
int ref_memory_per_gpu(const ref_plan* p, double nonexpert, double expert, double* out7) {
    return guarded([&] {
        ParallelPlan plan;
        plan.world_size = p->world_size;
        plan.expert_parallel = p->expert_parallel;
        plan.model_parallel = p->model_parallel;
        plan.zero_stage = p->zero_stage;
        plan.offload = p->offload != 0;
        const MemoryEstimate e = memory_per_gpu(plan, nonexpert, expert);
        const double v[7] = {e.nonexpert_params, e.expert_params, e.nonexpert_grads, e.expert_grads,
                             e.nonexpert_optim, e.expert_optim, e.gpu_total()};
        std::memcpy(out7, v, sizeof(v));
    });
}
int ref_max_model_size(const ref_plan* p, double budget, double base, double per_expert,
                       int64_t* max_experts, double* total) {
    return guarded([&] {
        ParallelPlan plan;
        plan.world_size = p->world_size;
        plan.expert_parallel = p->expert_parallel;
        plan.model_parallel = p->model_parallel;
        plan.zero_stage = p->zero_stage;
        plan.offload = p->offload != 0;
        const MaxModelSize m = max_model_size(plan, budget, base, per_expert);
        *max_experts = m.max_experts;
        *total = m.total_params;
    });
}

}  // extern "C"
