// plan.cpp — the reference's ZeRO-2 / expert-parallel memory planner
// (parallel.hpp:13-74, parallel.cpp:18-115) as the capacity check of the
// B200 layer.  Pure host arithmetic, same bytes-per-parameter model as the
// reference (kBytesParam 2 + kBytesGrad 2 + kBytesOptim 12, parallel.hpp:27-33),
// which is also this build's layout: bf16 parameters and gradients, fp32
// master weights and both Adam moments (optim.cu).
#include <cstdint>
#include <string>

#include "../../include/moe_b200.h"

namespace {

constexpr double kBytesParam = 2.0, kBytesGrad = 2.0, kBytesOptim = 12.0;

moe_status validate(const moe_parallel_plan* p, const char** why) {
    // ParallelPlan::validate, parallel.cpp:18-35
    if (!p) { *why = "plan: null"; return MOE_SHAPE; }
    if (p->world_size < 1 || p->expert_parallel < 1 || p->model_parallel < 1) {
        *why = "plan: all parallel degrees must be >= 1";
        return MOE_CONFIG;
    }
    if (p->zero_stage != 0 && p->zero_stage != 2) { *why = "plan: zero_stage must be 0 or 2"; return MOE_CONFIG; }
    if (p->world_size % p->model_parallel != 0) {
        *why = "plan: model_parallel must divide world_size";
        return MOE_CONFIG;
    }
    if (static_cast<long long>(p->model_parallel) * p->expert_parallel > p->world_size) {
        *why = "plan: model_parallel * expert_parallel exceeds world_size";
        return MOE_CONFIG;
    }
    if ((p->world_size / p->model_parallel) % p->expert_parallel != 0) {
        *why = "plan: expert_parallel must divide data_parallel";
        return MOE_CONFIG;
    }
    return MOE_OK;
}

void estimate(const moe_parallel_plan* p, double ne, double ex, moe_memory_estimate* e) {
    // memory_per_gpu, parallel.cpp:56-80
    const double mp = p->model_parallel, ep = p->expert_parallel;
    const double dp = static_cast<double>(p->world_size / p->model_parallel);
    const double ne_local = ne / mp, ex_local = ex / (ep * mp);
    const double ne_part = p->zero_stage == 2 ? dp : 1.0;
    const double ex_part = p->zero_stage == 2 ? dp / ep : 1.0;
    e->nonexpert_params = kBytesParam * ne_local;
    e->expert_params = kBytesParam * ex_local;
    e->nonexpert_grads = kBytesGrad * ne_local / ne_part;
    e->nonexpert_optim = kBytesOptim * ne_local / ne_part;
    e->expert_grads = kBytesGrad * ex_local / ex_part;
    e->expert_optim = kBytesOptim * ex_local / ex_part;
    e->grad_optim_on_cpu = p->offload ? 1 : 0;
    const double state = e->nonexpert_grads + e->expert_grads + e->nonexpert_optim + e->expert_optim;
    const double params = e->nonexpert_params + e->expert_params;
    e->gpu_total = params + (p->offload ? 0.0 : state);
    e->cpu_total = p->offload ? state : 0.0;
    e->optimizer_grad_share = state / (state + params);
}

thread_local std::string g_plan_err;

}  // namespace

extern "C" {

moe_status moe_plan_validate(const moe_parallel_plan* plan) {
    const char* why = "";
    const moe_status s = validate(plan, &why);
    g_plan_err = why;
    return s;
}

const char* moe_plan_last_error(void) { return g_plan_err.c_str(); }

moe_status moe_memory_per_gpu(const moe_parallel_plan* plan, double nonexpert_params,
                              double expert_params, moe_memory_estimate* out) {
    const char* why = "";
    moe_status s = validate(plan, &why);
    if (s == MOE_OK && (nonexpert_params < 0.0 || expert_params < 0.0)) {
        why = "memory_per_gpu: parameter counts must be >= 0";
        s = MOE_CONFIG;
    }
    if (s == MOE_OK && !out) { why = "memory_per_gpu: output required"; s = MOE_SHAPE; }
    g_plan_err = why;
    if (s == MOE_OK) estimate(plan, nonexpert_params, expert_params, out);
    return s;
}

moe_status moe_max_model_size(const moe_parallel_plan* plan, double gpu_budget_bytes, double base_params,
                              double params_per_expert, int64_t* max_experts, double* total_params) {
    // max_model_size, parallel.cpp:82-115 (monotone; doubling then bisection)
    const char* why = "";
    moe_status s = validate(plan, &why);
    if (s == MOE_OK && params_per_expert <= 0.0) {
        why = "max_model_size: params_per_expert must be positive";
        s = MOE_CONFIG;
    }
    moe_memory_estimate e{};
    if (s == MOE_OK) {
        estimate(plan, base_params, 0.0, &e);
        if (e.gpu_total > gpu_budget_bytes) {
            why = "max_model_size: base model alone exceeds the GPU budget";
            s = MOE_CONFIG;
        }
    }
    g_plan_err = why;
    if (s != MOE_OK) return s;
    auto fits = [&](int64_t n) {
        moe_memory_estimate m{};
        estimate(plan, base_params, params_per_expert * static_cast<double>(n), &m);
        return m.gpu_total <= gpu_budget_bytes;
    };
    int64_t hi = 1;
    while (fits(hi)) {
        hi *= 2;
        if (hi > (int64_t{1} << 50)) break;
    }
    int64_t lo = 0;
    while (lo + 1 < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (fits(mid)) lo = mid; else hi = mid;
    }
    if (max_experts) *max_experts = lo;
    if (total_params) *total_params = base_params + params_per_expert * static_cast<double>(lo);
    return MOE_OK;
}

}  // extern "C"
