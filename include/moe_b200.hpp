// moe_b200.hpp — C++ mirror of the reference's MoE-layer operator API
// (/root/reference/proj/core/include/moeforge/routing.hpp and parallel.hpp)
// over the C ABI of libmoe_b200.so (include/moe_b200.h).  Header-only.
//
// Same names and semantics as the reference: Phase, AssignmentMode,
// RouterConfig{...}.validate(), kDropped, RoutingDecision, capacity(),
// moe_layer_forward and the exception types of common.hpp (ShapeError,
// NonFiniteError, ConfigError, UniformShapeError) rethrown from moe_status.
// Tensors are device pointers; the reference's implicit tape backward becomes
// an explicit MoeLayer::backward on the saved context.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <utility>
#include <vector>

#include "moe_b200.h"

namespace moe_b200 {

// ---- errors (common.hpp:10-35) ----------------------------------------------
struct ShapeError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct NonFiniteError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ConfigError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct UniformShapeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(moe_status s, const moe_handle* h = nullptr, const char* what = "") {
    if (s == MOE_OK) return;
    std::string msg = h ? moe_last_error(h) : "";
    if (msg.empty()) msg = what;
    switch (s) {
        case MOE_SHAPE: throw ShapeError(msg);
        case MOE_CONFIG: throw ConfigError(msg);
        case MOE_NONFINITE: throw NonFiniteError(msg);
        case MOE_UNIFORM_SHAPE: throw UniformShapeError(msg);
        case MOE_INVALID_ARG: throw std::invalid_argument(msg);
        default: throw CudaError(msg);
    }
}

enum class Phase { kTrain = MOE_TRAIN, kEval = MOE_EVAL };                  // routing.hpp:13
enum class AssignmentMode { kPlain = MOE_PLAIN, kGrouped = MOE_GROUPED, kRts = MOE_RTS };

struct RouterConfig {  // routing.hpp:17-32
    int num_experts = 8;
    double capacity_factor_train = 1.0;
    double capacity_factor_eval = 2.0;
    double jitter_eps = 0.01;
    double balance_coeff = 0.01;
    AssignmentMode assignment_mode = AssignmentMode::kPlain;
    int group_count = 1;
    int top_k = 1;
    std::uint64_t rng_seed = 0;

    moe_router_cfg c() const {
        return moe_router_cfg{num_experts, capacity_factor_train, capacity_factor_eval, jitter_eps,
                              balance_coeff, static_cast<int>(assignment_mode), group_count, top_k,
                              rng_seed};
    }
    void validate() const {
        const moe_router_cfg cc = c();
        check(moe_router_cfg_validate(&cc), nullptr, "router: invalid config");
    }
    double capacity_factor(Phase phase) const {
        return phase == Phase::kTrain ? capacity_factor_train : capacity_factor_eval;
    }
};

inline constexpr std::int32_t kDropped = MOE_KDROPPED;  // routing.hpp:34

// routing.cpp:43-49
inline int capacity(std::int64_t tokens, const RouterConfig& cfg, Phase phase) {
    const moe_router_cfg cc = cfg.c();
    int cap = 0;
    check(moe_capacity(tokens, &cc, static_cast<int>(phase), &cap), nullptr,
          "capacity: token count must be >= 1");
    return cap;
}

inline std::uint64_t derive_seed(std::uint64_t seed, const char* tag) {
    return moe_derive_seed_tag(seed, tag);
}
inline std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t salt) {
    return moe_derive_seed_u64(seed, salt);
}

// RoutingDecision (routing.hpp:38-57) copied to the host.
struct RoutingDecision {
    int num_experts = 0;
    int capacity = 0;
    int top_k = 1;
    std::vector<std::int32_t> expert_id;
    std::vector<std::int32_t> slot;
    std::vector<float> gate_prob;

    std::int64_t tokens() const { return static_cast<std::int64_t>(expert_id.size()) / top_k; }
    bool kept(std::int64_t token, int k = 0) const { return slot[token * top_k + k] != kDropped; }
    std::int64_t drop_count() const {
        std::int64_t n = 0;
        for (auto s : slot) n += s == kDropped;
        return n;
    }
    std::vector<std::int64_t> kept_per_expert() const {
        std::vector<std::int64_t> c(static_cast<size_t>(num_experts), 0);
        for (size_t i = 0; i < slot.size(); ++i)
            if (slot[i] != kDropped) ++c[static_cast<size_t>(expert_id[i])];
        return c;
    }
};

// Device-resident layer parameters in the reference orientation, packed per
// expert: gate_w [d,E]; w1 [E_local,d,f]; b1 [E_local,f]; w2 [E_local,f,d]; b2 [E_local,d].
struct MoeLayerParams {
    const float* gate_w = nullptr;
    const void* w1 = nullptr;
    const float* b1 = nullptr;
    const void* w2 = nullptr;
    const float* b2 = nullptr;
};

struct MoeLayerGrads {  // written (not accumulated) by backward
    void* dx = nullptr;
    float* dgate_w = nullptr;
    void* dw1 = nullptr;
    float* db1 = nullptr;
    void* dw2 = nullptr;
    float* db2 = nullptr;
    void* dresidual = nullptr;  // only when forward got a residual
};

// One layer instance: workspace + saved forward context on one stream.
class MoeLayer {
public:
    MoeLayer(const RouterConfig& cfg, std::int64_t max_tokens, std::int64_t d_model,
             std::int64_t d_ff, moe_dtype dtype = MOE_BF16, int ep_size = 1, int ep_rank = 0)
        : cfg_(cfg) {
        const moe_router_cfg cc = cfg.c();
        const moe_layer_dims dims{max_tokens, d_model, d_ff, dtype, ep_size, ep_rank};
        check(moe_create(&cc, &dims, &h_), nullptr, "moe_create failed");
    }
    ~MoeLayer() { moe_destroy(h_); }
    MoeLayer(const MoeLayer&) = delete;
    MoeLayer& operator=(const MoeLayer&) = delete;

    void set_stream(cudaStream_t s) { check(moe_set_stream(h_, s), h_); }
    // parallel.hpp:100-111 made physical: bind to an NCCL communicator
    void ep_init(const void* nccl_unique_id) { check(moe_ep_init(h_, nccl_unique_id), h_); }

    // moe_layer_forward (routing.hpp:144-147).  residual == nullptr means x.
    // aux is one device float.  Decision outputs are optional device arrays.
    void forward(std::int64_t T, const void* x, const MoeLayerParams& p, Phase phase,
                 std::uint64_t seed, void* y, float* aux, const void* residual = nullptr,
                 std::int32_t* expert_id = nullptr, std::int32_t* slot = nullptr,
                 float* gate_prob = nullptr, bool check_flags = true) {
        check(moe_forward(h_, T, x, p.gate_w, p.w1, p.b1, p.w2, p.b2, static_cast<int>(phase), seed,
                          residual, y, aux, expert_id, slot, gate_prob),
              h_);
        if (check_flags) sync_check();
    }
    // Backward of <dy, y> + daux * aux (the reference tape, tensor.cpp:156-187).
    void backward(const void* dy, float daux, const MoeLayerGrads& g, bool check_flags = true) {
        check(moe_backward(h_, dy, daux, g.dx, g.dgate_w, g.dw1, g.db1, g.dw2, g.db2, g.dresidual), h_);
        if (check_flags) sync_check();
    }
    void sync_check() { check(moe_check(h_, nullptr), h_); }

    // RoutingDecision of the last forward, on the host.
    RoutingDecision decision(std::int64_t T, const std::int32_t* expert_id_dev,
                             const std::int32_t* slot_dev, const float* gate_prob_dev) {
        RoutingDecision d;
        d.num_experts = cfg_.num_experts;
        d.top_k = cfg_.top_k;
        std::int64_t drops = 0;
        check(moe_last_decision_stats(h_, &d.capacity, &drops, nullptr), h_);
        const size_t n = static_cast<size_t>(T * cfg_.top_k);
        d.expert_id.resize(n);
        d.slot.resize(n);
        d.gate_prob.resize(n);
        cudaMemcpy(d.expert_id.data(), expert_id_dev, 4 * n, cudaMemcpyDeviceToHost);
        cudaMemcpy(d.slot.data(), slot_dev, 4 * n, cudaMemcpyDeviceToHost);
        cudaMemcpy(d.gate_prob.data(), gate_prob_dev, 4 * n, cudaMemcpyDeviceToHost);
        return d;
    }

    moe_handle* handle() const { return h_; }
    const RouterConfig& config() const { return cfg_; }

private:
    RouterConfig cfg_;
    moe_handle* h_ = nullptr;
};

// ---- per-stage operators (routing.hpp:60-118) --------------------------------
// Same names and semantics as the reference; tensors are device buffers owned
// by DeviceArray (RAII), decisions are host RoutingDecision values as in the
// reference.  Each call runs on the legacy default stream through a scratch
// handle cached per (config, d_model, dtype) and synchronises before it returns.
template <class T>
class DeviceArray {
public:
    DeviceArray() = default;
    explicit DeviceArray(size_t n) : n_(n) {
        if (cudaMalloc(&p_, sizeof(T) * (n ? n : 1)) != cudaSuccess) throw CudaError("cudaMalloc failed");
    }
    DeviceArray(const std::vector<T>& host) : DeviceArray(host.size()) {
        cudaMemcpy(p_, host.data(), sizeof(T) * n_, cudaMemcpyHostToDevice);
    }
    ~DeviceArray() { cudaFree(p_); }
    DeviceArray(DeviceArray&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
    DeviceArray& operator=(DeviceArray&& o) noexcept {
        std::swap(p_, o.p_);
        std::swap(n_, o.n_);
        return *this;
    }
    DeviceArray(const DeviceArray&) = delete;
    T* data() const { return p_; }
    size_t size() const { return n_; }
    std::vector<T> to_host() const {
        std::vector<T> h(n_);
        cudaMemcpy(h.data(), p_, sizeof(T) * n_, cudaMemcpyDeviceToHost);
        return h;
    }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
};

namespace detail {
struct HandleDel {
    void operator()(moe_handle* h) const { moe_destroy(h); }
};
// scratch handle with >= T tokens, d_model d, dtype, and room for `cap` slots
inline moe_handle* scratch(const RouterConfig& cfg, std::int64_t T, std::int64_t d, moe_dtype dt, int cap = 0) {
    using Key = std::tuple<int, int, int, double, double, double, double, std::int64_t, int>;
    static std::map<Key, std::tuple<std::unique_ptr<moe_handle, HandleDel>, std::int64_t, int>> cache;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    const Key key{cfg.num_experts, cfg.top_k, cfg.group_count, cfg.capacity_factor_train,
                  cfg.capacity_factor_eval, cfg.jitter_eps, cfg.balance_coeff, d, static_cast<int>(dt)};
    auto& e = cache[key];
    if (!std::get<0>(e) || std::get<1>(e) < T || std::get<2>(e) < cap) {
        const std::int64_t Tn = std::max(T, std::get<1>(e));
        const int capn = std::max(cap, std::get<2>(e));
        moe_router_cfg c = cfg.c();
        c.capacity_factor_eval = std::max(c.capacity_factor_eval,
                                          static_cast<double>(capn) * cfg.num_experts / static_cast<double>(Tn) + 1.0);
        const moe_layer_dims dims{Tn, d, 8, dt, 1, 0};
        moe_handle* h = nullptr;
        check(moe_create(&c, &dims, &h), nullptr, "moe_create (per-stage scratch)");
        std::get<0>(e).reset(h);
        std::get<1>(e) = Tn;
        std::get<2>(e) = capn;
    }
    return std::get<0>(e).get();
}
inline void sync(moe_handle* h) { check(moe_check(h, nullptr), h); }
}  // namespace detail

struct GateResult {  // routing.hpp:62-66
    DeviceArray<float> probs;                  // [T, E]
    std::vector<std::int32_t> choice;          // [T * top_k], ties to the lowest index
    std::vector<DeviceArray<float>> gate_prob;  // per k: [T]
};

// routing.cpp:51-101; x is [T, d] of dtype (MOE_F32 / MOE_BF16), gate_w [d, E] fp32
inline GateResult gate_forward(const void* x, std::int64_t T, std::int64_t d, moe_dtype dtype, const float* gate_w,
                               const RouterConfig& cfg, Phase phase, std::uint64_t jitter_seed) {
    cfg.validate();
    const int E = cfg.num_experts, K = cfg.top_k;
    moe_handle* h = detail::scratch(cfg, T, d, dtype);
    GateResult g{DeviceArray<float>(static_cast<size_t>(T * E)), {}, {}};
    DeviceArray<std::int32_t> ch(static_cast<size_t>(T * K));
    DeviceArray<float> gp(static_cast<size_t>(T * K));
    check(moe_gate(h, T, x, gate_w, static_cast<int>(phase), jitter_seed, g.probs.data(), ch.data(), gp.data()), h);
    detail::sync(h);
    g.choice = ch.to_host();
    const std::vector<float> all = gp.to_host();
    for (int k = 0; k < K; ++k) {
        std::vector<float> col(static_cast<size_t>(T));
        for (std::int64_t t = 0; t < T; ++t) col[static_cast<size_t>(t)] = all[static_cast<size_t>(t * K + k)];
        g.gate_prob.emplace_back(col);
    }
    return g;
}

namespace detail {
inline RoutingDecision assign(const std::vector<std::int32_t>& choice, int E, int cap, int K, int mode, int G,
                              std::uint64_t seed) {
    RoutingDecision dec;
    dec.num_experts = E;
    dec.top_k = K;
    dec.expert_id = choice;
    dec.slot.assign(choice.size(), kDropped);
    dec.gate_prob.assign(choice.size(), 0.f);
    const std::int64_t T = static_cast<std::int64_t>(choice.size()) / K;
    dec.capacity = mode == MOE_GROUPED ? G * ((cap + G - 1) / G) : cap;
    if (T == 0) return dec;
    RouterConfig c;
    c.num_experts = E;
    c.top_k = K;
    c.group_count = mode == MOE_GROUPED ? G : 1;
    moe_handle* h = scratch(c, T, 8, MOE_F32, cap);
    DeviceArray<std::int32_t> ch(choice), sl(choice.size());
    int cap_out = 0;
    check(moe_assign_mode(h, T, ch.data(), cap, mode, G, seed, sl.data(), &cap_out), h);
    dec.slot = sl.to_host();
    dec.capacity = cap_out;
    return dec;
}
}  // namespace detail

// routing.cpp:147-206 (k-major order-dependent scans; capacity ignores top_k)
inline RoutingDecision assign_plain(const std::vector<std::int32_t>& choice, int num_experts, int cap, int top_k = 1) {
    return detail::assign(choice, num_experts, cap, top_k, MOE_PLAIN, 1, 0);
}
inline RoutingDecision assign_grouped(const std::vector<std::int32_t>& choice, int num_experts, int cap,
                                      int group_count, int top_k = 1) {
    return detail::assign(choice, num_experts, cap, top_k, MOE_GROUPED, group_count, 0);
}
inline RoutingDecision assign_rts(const std::vector<std::int32_t>& choice, int num_experts, int cap,
                                  std::uint64_t rng_seed, int top_k = 1) {
    return detail::assign(choice, num_experts, cap, top_k, MOE_RTS, 1, rng_seed);
}
inline RoutingDecision make_assignment(const std::vector<std::int32_t>& choice, std::int64_t tokens,
                                       const RouterConfig& cfg, Phase phase, std::uint64_t rng_seed) {
    const int cap = capacity(tokens, cfg, phase);
    if (phase == Phase::kEval) return assign_plain(choice, cfg.num_experts, cap, cfg.top_k);
    switch (cfg.assignment_mode) {
        case AssignmentMode::kPlain: return assign_plain(choice, cfg.num_experts, cap, cfg.top_k);
        case AssignmentMode::kGrouped:
            return assign_grouped(choice, cfg.num_experts, cap, cfg.group_count, cfg.top_k);
        case AssignmentMode::kRts: return assign_rts(choice, cfg.num_experts, cap, rng_seed, cfg.top_k);
    }
    throw ConfigError("make_assignment: unknown mode");
}

struct DispatchBuffer {  // routing.hpp:96-104
    DeviceArray<std::uint8_t> data;       // [E * capacity, d] of the activation dtype
    int num_experts = 0;
    int capacity = 0;
    DeviceArray<std::uint8_t> occupancy;  // [E * capacity]
};

// routing.cpp:208-243: kept rows scattered to row e * capacity + slot, other rows zero
inline DispatchBuffer dispatch(const void* x, std::int64_t T, std::int64_t d, moe_dtype dtype,
                               const RoutingDecision& dec) {
    RouterConfig c;
    c.num_experts = dec.num_experts;
    c.top_k = dec.top_k;
    moe_handle* h = detail::scratch(c, T, d, dtype);
    const size_t rows = static_cast<size_t>(dec.num_experts) * dec.capacity;
    const size_t es = dtype == MOE_BF16 ? 2 : 4;
    DispatchBuffer b{DeviceArray<std::uint8_t>(rows * d * es), dec.num_experts, dec.capacity,
                     DeviceArray<std::uint8_t>(rows)};
    DeviceArray<std::int32_t> eid(dec.expert_id), sl(dec.slot);
    check(moe_dispatch(h, T, x, eid.data(), sl.data(), dec.capacity, b.data.data(), b.occupancy.data()), h);
    detail::sync(h);
    return b;
}

// routing.cpp:258-298: y[t] = sum_{k kept} weights[k][t] * out[row(t,k)], else residual[t];
// weights: [top_k][T] fp32 device
inline DeviceArray<std::uint8_t> combine(const void* expert_out, std::int64_t d, moe_dtype dtype,
                                         const RoutingDecision& dec, const void* residual, const float* weights) {
    const std::int64_t T = dec.tokens();
    RouterConfig c;
    c.num_experts = dec.num_experts;
    c.top_k = dec.top_k;
    moe_handle* h = detail::scratch(c, T, d, dtype);
    const size_t es = dtype == MOE_BF16 ? 2 : 4;
    DeviceArray<std::uint8_t> y(static_cast<size_t>(T * d) * es);
    DeviceArray<std::int32_t> eid(dec.expert_id), sl(dec.slot);
    check(moe_combine(h, T, expert_out, eid.data(), sl.data(), dec.capacity, residual, weights, y.data()), h);
    detail::sync(h);
    return y;
}

// routing.cpp:348-374: alpha * E * sum_e f_e * mean_t P[t, e] (first choices, drops
// included); rows of probs must sum to 1 (else std::invalid_argument)
inline float balance_loss(const float* probs, const RoutingDecision& dec, double alpha) {
    const std::int64_t T = dec.tokens();
    RouterConfig c;
    c.num_experts = dec.num_experts;
    c.top_k = dec.top_k;
    moe_handle* h = detail::scratch(c, T, 8, MOE_F32);
    DeviceArray<std::int32_t> eid(dec.expert_id);
    DeviceArray<float> out(1);
    check(moe_balance_loss(h, T, probs, eid.data(), alpha, out.data()), h);
    return out.to_host()[0];
}

// moe_layer_forward (routing.hpp:144-147) on a layer instance: writes y / aux
// (device) and returns the RoutingDecision; layer.backward() is the tape's pass.
inline RoutingDecision moe_layer_forward(MoeLayer& layer, std::int64_t T, const void* x, const MoeLayerParams& p,
                                         Phase phase, std::uint64_t seed, void* y, float* aux,
                                         const void* residual = nullptr) {
    const int K = layer.config().top_k;
    DeviceArray<std::int32_t> eid(static_cast<size_t>(T * K)), sl(static_cast<size_t>(T * K));
    DeviceArray<float> gp(static_cast<size_t>(T * K));
    layer.forward(T, x, p, phase, seed, y, aux, residual, eid.data(), sl.data(), gp.data());
    return layer.decision(T, eid.data(), sl.data(), gp.data());
}

}  // namespace moe_b200
