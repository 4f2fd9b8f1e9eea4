// routing_b200.cpp — the drop-in: the reference's MoE operator API
// (moeforge/routing.hpp) implemented on libmoe_b200.so, compiled against the
// reference's own headers and Tensor.  A maintainer adds
// this file to core/CMakeLists.txt in place of the routing.cpp definitions
// it replaces; every caller — run_moe (model.cpp:340-350), the trainer,
// gradcheck (tests/support/gradcheck.hpp:28-57) — is unchanged.
//
// Replaced here (the rest of routing.cpp — RouterConfig::validate,
// RoutingDecision, capacity, gate_forward, dispatch, combine, balance_loss —
// stays the reference's):
//
//   moe_layer_forward (routing.cpp:376-424)  one tape node for y and one for
//       aux_loss over the device float64 path (moe_forward_f64); the nodes'
//       closures run moe_backward_f64 and add (+=, tensor.cpp:31-36) into the
//       parents' grads, so Tensor::backward() (tensor.cpp:156-187) drives the
//       device backward exactly where the reference's closures would run;
//   assign_plain / assign_grouped / assign_rts / make_assignment
//       (routing.cpp:147-206) on the device assignment scan (moe_assign_mode).
//
// Errors come back as the reference's exception types (common.hpp:10-35).
#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "moeforge/common.hpp"
#include "moeforge/routing.hpp"
#include "moeforge/tensor.hpp"
#include "moe_b200.h"

namespace moeforge {

namespace {

[[noreturn]] void rethrow(moe_status s, const std::string& what) {
    switch (s) {
        case MOE_SHAPE: throw ShapeError(what);
        case MOE_CONFIG: throw ConfigError(what);
        case MOE_NONFINITE: throw NonFiniteError(what);
        case MOE_UNIFORM_SHAPE: throw UniformShapeError(what);
        case MOE_INVALID_ARG: throw std::invalid_argument(what);
        default: throw std::runtime_error("libmoe_b200: " + what);
    }
}
void ok(moe_status s, const moe_handle* h, const char* what) {
    if (s == MOE_OK) return;
    std::string m = h ? moe_last_error(h) : "";
    rethrow(s, m.empty() ? std::string(what) : m);
}
void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

moe_router_cfg to_c(const RouterConfig& c) {
    moe_router_cfg r{};
    r.num_experts = c.num_experts;
    r.capacity_factor_train = c.capacity_factor_train;
    r.capacity_factor_eval = c.capacity_factor_eval;
    r.jitter_eps = c.jitter_eps;
    r.balance_coeff = c.balance_coeff;
    r.assignment_mode = static_cast<int>(c.assignment_mode);
    r.group_count = c.group_count;
    r.top_k = c.top_k;
    r.rng_seed = c.rng_seed;
    return r;
}

// RAII device buffer
struct Dev {
    void* p = nullptr;
    size_t bytes = 0;
    explicit Dev(size_t n) : bytes(n ? n : 16) { cuda_ok(cudaMalloc(&p, bytes), "cudaMalloc"); }
    ~Dev() { cudaFree(p); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    double* d() const { return static_cast<double*>(p); }
    int32_t* i() const { return static_cast<int32_t*>(p); }
    void up(const void* src, size_t n) { cuda_ok(cudaMemcpy(p, src, n, cudaMemcpyHostToDevice), "upload"); }
    void down(void* dst, size_t n) const { cuda_ok(cudaMemcpy(dst, p, n, cudaMemcpyDeviceToHost), "download"); }
};

struct HandleDel {
    void operator()(moe_handle* h) const { moe_destroy(h); }
};
using Handle = std::unique_ptr<moe_handle, HandleDel>;

// One moe_layer_forward call on the device: its handle keeps the forward
// context; the output nodes' closures call backward() (y with daux = 0, aux
// with dy = 0 — the layer is linear in (dy, daux), so the two calls sum to
// the reference's single pass).
struct LayerCall {
    Handle h;
    int64_t T = 0, d = 0, f = 0;
    int E = 0;
    std::unique_ptr<Dev> x, gw, w1, b1, w2, b2, res, y, aux, eid, slot, gp;
    std::vector<std::shared_ptr<Tensor::Node>> parents;  // x, gate_w, experts..., residual?
    bool has_res = false;

    void backward(const double* dy_host, double daux) {
        const size_t Td = static_cast<size_t>(T * d);
        Dev dy(8 * Td), dx(8 * Td), dgw(8 * d * E), dw1(8 * E * d * f), db1(8 * E * f), dw2(8 * E * f * d),
            db2(8 * E * d), dres(8 * Td);
        if (dy_host) dy.up(dy_host, 8 * Td);
        else cuda_ok(cudaMemset(dy.p, 0, 8 * Td), "memset");
        ok(moe_backward_f64(h.get(), dy.d(), daux, dx.d(), dgw.d(), dw1.d(), db1.d(), dw2.d(), db2.d(),
                            has_res ? dres.d() : nullptr, 0),
           h.get(), "moe_backward_f64");
        ok(moe_check(h.get(), nullptr), h.get(), "moe_backward_f64");
        auto add_into = [](const std::shared_ptr<Tensor::Node>& n, const Dev& src, size_t off_elems) {
            if (!n->requires_grad) return;
            std::vector<double> v(n->value.size());
            cuda_ok(cudaMemcpy(v.data(), src.d() + off_elems, 8 * v.size(), cudaMemcpyDeviceToHost), "download");
            auto g = n->ensure_grad();
            for (size_t i = 0; i < v.size(); ++i) g[i] += v[i];
        };
        add_into(parents[0], dx, 0);
        add_into(parents[1], dgw, 0);
        for (int e = 0; e < E; ++e) {
            add_into(parents[2 + 4 * e + 0], dw1, static_cast<size_t>(e) * d * f);
            add_into(parents[2 + 4 * e + 1], db1, static_cast<size_t>(e) * f);
            add_into(parents[2 + 4 * e + 2], dw2, static_cast<size_t>(e) * f * d);
            add_into(parents[2 + 4 * e + 3], db2, static_cast<size_t>(e) * d);
        }
        if (has_res) add_into(parents.back(), dres, 0);
    }
};

std::vector<double> pack(const std::vector<ExpertFfn>& ex, Tensor ExpertFfn::*m) {
    std::vector<double> out;
    for (const ExpertFfn& e : ex) {
        auto v = (e.*m).data();
        out.insert(out.end(), v.begin(), v.end());
    }
    return out;
}

// A cached device handle for the assignment scans (grown on demand).
struct AssignCache {
    std::mutex mu;
    std::map<std::tuple<int, int, int>, std::tuple<Handle, int64_t, int>> by_shape;  // (E,K,G) -> (h, T, cap)
};
AssignCache& assign_cache() {
    static AssignCache c;
    return c;
}

RoutingDecision device_assign(std::span<const std::int32_t> choice, int num_experts, int cap, int top_k,
                              int mode, int group_count, std::uint64_t seed) {
    // routing.cpp:105-111 range check on the host first (same message)
    for (std::int32_t c : choice)
        if (c < 0 || c >= num_experts) throw ConfigError("assignment: choice out of expert range");
    const int64_t T = static_cast<int64_t>(choice.size()) / top_k;
    if (mode == MOE_GROUPED && (group_count < 1 || T % group_count != 0))
        throw ConfigError("assign_grouped: group_count must divide the token count");
    RoutingDecision dec;
    dec.num_experts = num_experts;
    dec.top_k = top_k;
    dec.expert_id.assign(choice.begin(), choice.end());
    dec.slot.assign(choice.size(), kDropped);
    dec.gate_prob.assign(choice.size(), 0.0);
    const int G = mode == MOE_GROUPED ? group_count : 1;
    dec.capacity = mode == MOE_GROUPED ? G * ((cap + G - 1) / G) : cap;
    if (T == 0) return dec;
    AssignCache& ac = assign_cache();
    std::lock_guard<std::mutex> lk(ac.mu);
    auto& slot = ac.by_shape[{num_experts, top_k, G}];
    Handle& h = std::get<0>(slot);
    if (!h || std::get<1>(slot) < T || std::get<2>(slot) < cap) {
        const int64_t Tn = std::max<int64_t>(T, std::get<1>(slot));
        const int capn = std::max(cap, std::get<2>(slot));
        moe_router_cfg c{};
        moe_router_cfg_default(&c);
        c.num_experts = num_experts;
        c.top_k = top_k;
        c.group_count = G;
        // eval-phase capacity sized so the workspace holds `capn` slots per expert
        c.capacity_factor_eval = static_cast<double>(capn) * num_experts / static_cast<double>(Tn) + 1.0;
        const moe_layer_dims dims{Tn, 8, 8, MOE_F32, 1, 0};
        moe_handle* raw = nullptr;
        ok(moe_create(&c, &dims, &raw), nullptr, "moe_create (assignment scratch)");
        h.reset(raw);
        std::get<1>(slot) = Tn;
        std::get<2>(slot) = capn;
    }
    Dev dch(4 * choice.size()), dsl(4 * choice.size());
    dch.up(choice.data(), 4 * choice.size());
    int cap_out = 0;
    ok(moe_assign_mode(h.get(), T, dch.i(), cap, mode, G, seed, dsl.i(), &cap_out), h.get(), "assign");
    dsl.down(dec.slot.data(), 4 * choice.size());
    dec.capacity = cap_out;
    return dec;
}

}  // namespace

// ---- assignment (routing.cpp:147-206) on the device scan -------------------
RoutingDecision assign_plain(std::span<const std::int32_t> choice, int num_experts, int cap, int top_k) {
    return device_assign(choice, num_experts, cap, top_k, MOE_PLAIN, 1, 0);
}

RoutingDecision assign_grouped(std::span<const std::int32_t> choice, int num_experts, int cap,
                               int group_count, int top_k) {
    return device_assign(choice, num_experts, cap, top_k, MOE_GROUPED, group_count, 0);
}

RoutingDecision assign_rts(std::span<const std::int32_t> choice, int num_experts, int cap,
                           std::uint64_t rng_seed, int top_k) {
    return device_assign(choice, num_experts, cap, top_k, MOE_RTS, 1, rng_seed);
}

RoutingDecision make_assignment(std::span<const std::int32_t> choice, std::int64_t tokens,
                                const RouterConfig& cfg, Phase phase, std::uint64_t rng_seed) {
    const int cap = capacity(tokens, cfg, phase);
    if (phase == Phase::kEval) return assign_plain(choice, cfg.num_experts, cap, cfg.top_k);  // routing.cpp:194-196
    switch (cfg.assignment_mode) {
        case AssignmentMode::kPlain: return assign_plain(choice, cfg.num_experts, cap, cfg.top_k);
        case AssignmentMode::kGrouped:
            return assign_grouped(choice, cfg.num_experts, cap, cfg.group_count, cfg.top_k);
        case AssignmentMode::kRts: return assign_rts(choice, cfg.num_experts, cap, rng_seed, cfg.top_k);
    }
    throw ConfigError("make_assignment: unknown mode");
}

// ---- moe_layer_forward (routing.cpp:376-424) on the device f64 path --------
MoeLayerResult moe_layer_forward(const Tensor& x, const MoeLayerParams& params, const RouterConfig& cfg,
                                 Phase phase, std::uint64_t seed, const Tensor* residual) {
    cfg.validate();
    if (static_cast<int>(params.experts.size()) != cfg.num_experts)
        throw ShapeError("moe_layer_forward: expert count does not match config");
    if (x.shape().size() != 2 || params.gate_w.shape().size() != 2 || x.shape()[1] != params.gate_w.shape()[0] ||
        params.gate_w.shape()[1] != cfg.num_experts)
        throw ShapeError("gate_forward: x [T,d] and gate_w [d,E] required");
    auto call = std::make_shared<LayerCall>();
    call->T = x.shape()[0];
    call->d = x.shape()[1];
    call->E = cfg.num_experts;
    const int64_t T = call->T, d = call->d;
    const int E = call->E, K = cfg.top_k;
    const ExpertFfn& e0 = params.experts[0];
    if (e0.w1.shape().size() != 2 || e0.w1.shape()[0] != d)
        throw ShapeError("matmul: inner dimensions do not match");
    const int64_t f = e0.w1.shape()[1];
    call->f = f;
    for (const ExpertFfn& e : params.experts)
        if (e.w1.shape() != std::vector<int64_t>{d, f} || e.w2.shape() != std::vector<int64_t>{f, d} ||
            e.b1.numel() != f || e.b2.numel() != d)
            throw ShapeError("moe_layer_forward: expert shapes differ");
    if (residual && residual->shape() != x.shape()) throw ShapeError("combine: residual must be [T, d]");

    const moe_router_cfg c = to_c(cfg);
    const moe_layer_dims dims{T, d, f, MOE_F64, 1, 0};
    moe_handle* raw = nullptr;
    ok(moe_create(&c, &dims, &raw), nullptr, "moe_create");
    call->h.reset(raw);
    auto up = [](std::unique_ptr<Dev>& dst, std::span<const double> v) {
        dst = std::make_unique<Dev>(8 * v.size());
        dst->up(v.data(), 8 * v.size());
    };
    up(call->x, x.data());
    up(call->gw, params.gate_w.data());
    const std::vector<double> W1 = pack(params.experts, &ExpertFfn::w1), B1 = pack(params.experts, &ExpertFfn::b1),
                              W2 = pack(params.experts, &ExpertFfn::w2), B2 = pack(params.experts, &ExpertFfn::b2);
    up(call->w1, W1);
    up(call->b1, B1);
    up(call->w2, W2);
    up(call->b2, B2);
    if (residual) up(call->res, residual->data());
    call->has_res = residual != nullptr;
    call->y = std::make_unique<Dev>(8 * T * d);
    call->aux = std::make_unique<Dev>(8);
    call->eid = std::make_unique<Dev>(4 * T * K);
    call->slot = std::make_unique<Dev>(4 * T * K);
    call->gp = std::make_unique<Dev>(8 * T * K);
    ok(moe_forward_f64(call->h.get(), T, call->x->d(), call->gw->d(), call->w1->d(), call->b1->d(), call->w2->d(),
                       call->b2->d(), phase == Phase::kTrain ? MOE_TRAIN : MOE_EVAL, seed,
                       residual ? call->res->d() : nullptr, call->y->d(), call->aux->d(), call->eid->i(),
                       call->slot->i(), call->gp->d()),
       call->h.get(), "moe_forward_f64");
    ok(moe_check(call->h.get(), nullptr), call->h.get(), "moe_forward_f64");

    std::vector<double> yv(static_cast<size_t>(T * d));
    double auxv = 0.0;
    call->y->down(yv.data(), 8 * yv.size());
    call->aux->down(&auxv, 8);
    MoeLayerResult out;
    RoutingDecision& dec = out.decision;
    dec.num_experts = E;
    dec.top_k = K;
    dec.expert_id.resize(static_cast<size_t>(T * K));
    dec.slot.resize(static_cast<size_t>(T * K));
    dec.gate_prob.resize(static_cast<size_t>(T * K));
    call->eid->down(dec.expert_id.data(), 4 * dec.expert_id.size());
    call->slot->down(dec.slot.data(), 4 * dec.slot.size());
    call->gp->down(dec.gate_prob.data(), 8 * dec.gate_prob.size());
    int cap = 0;
    ok(moe_last_decision_stats(call->h.get(), &cap, nullptr, nullptr), call->h.get(), "decision stats");
    dec.capacity = cap;

    // one tape node per output, inputs in a fixed order (LayerCall::parents)
    std::vector<Tensor> inputs = {x, params.gate_w};
    for (const ExpertFfn& e : params.experts) inputs.insert(inputs.end(), {e.w1, e.b1, e.w2, e.b2});
    if (residual) inputs.push_back(*residual);
    for (const Tensor& t : inputs) call->parents.push_back(t.node_ptr());
    out.y = Tensor::from_op({T, d}, std::move(yv), inputs,
                            [call](Tensor::Node& self) { call->backward(self.grad.data(), 0.0); }, "moe_b200");
    out.aux_loss = Tensor::from_op({1}, {auxv}, inputs,
                                   [call](Tensor::Node& self) { call->backward(nullptr, self.grad[0]); },
                                   "moe_b200_balance_loss");
    return out;
}

}  // namespace moeforge
