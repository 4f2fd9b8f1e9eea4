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

}  // namespace moe_b200
