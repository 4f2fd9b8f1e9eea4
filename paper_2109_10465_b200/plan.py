"""Capacity check of a training plan: the reference's
ZeRO-2 / expert-parallel memory planner (parallel.hpp:13-74,
parallel.cpp:18-115) over the C ABI, plus the layer workspace the B200
handles really allocate.

``memory_per_gpu`` / ``max_model_size`` keep the reference's names, fields and
ConfigError behaviour; ``capacity_check`` is the B200 addition: parameter
state from the planner + every handle's measured workspace against the
device's HBM, raising ConfigError when the plan does not fit.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _lib as L
from .routing import ConfigError, MoeError, ShapeError

_EXC = {L.MOE_CONFIG: ConfigError, L.MOE_SHAPE: ShapeError}

# parallel.hpp:27-33 (also this build's layout: bf16 param + grad, fp32 master + m + v)
K_BYTES_PARAM, K_BYTES_GRAD, K_BYTES_OPTIM = 2.0, 2.0, 12.0


@dataclass
class ParallelPlan:  # parallel.hpp:13-24
    world_size: int = 1
    expert_parallel: int = 1
    model_parallel: int = 1
    zero_stage: int = 0
    offload: bool = False

    def data_parallel(self) -> int:
        return self.world_size // self.model_parallel

    def to_c(self):
        return L.moe_parallel_plan(self.world_size, self.expert_parallel, self.model_parallel,
                                   self.zero_stage, int(self.offload))

    def validate(self) -> None:
        c = self.to_c()
        _raise(L.load().moe_plan_validate(C.byref(c)))


@dataclass
class MemoryEstimate:  # parallel.hpp:35-54 (bytes)
    nonexpert_params: float
    expert_params: float
    nonexpert_grads: float
    expert_grads: float
    nonexpert_optim: float
    expert_optim: float
    grad_optim_on_cpu: bool
    gpu: float
    cpu: float
    share: float

    def gpu_total(self) -> float:
        return self.gpu

    def cpu_total(self) -> float:
        return self.cpu

    def total(self) -> float:
        return self.gpu + self.cpu

    def optimizer_grad_share(self) -> float:
        return self.share


def _raise(st: int) -> None:
    if st != L.MOE_OK:
        msg = L.load().moe_plan_last_error().decode()
        raise _EXC.get(st, MoeError)(msg)


def memory_per_gpu(plan: ParallelPlan, nonexpert_params: float, expert_params: float) -> MemoryEstimate:
    """parallel.cpp:56-80: non-expert state sliced by mp and (stage 2)
    partitioned across dp; expert state sliced by ep*mp and partitioned across
    dp/ep; offload moves grads + optimizer to the host."""
    c = plan.to_c()
    e = L.moe_memory_estimate()
    _raise(L.load().moe_memory_per_gpu(C.byref(c), float(nonexpert_params), float(expert_params),
                                       C.byref(e)))
    return MemoryEstimate(e.nonexpert_params, e.expert_params, e.nonexpert_grads, e.expert_grads,
                          e.nonexpert_optim, e.expert_optim, bool(e.grad_optim_on_cpu), e.gpu_total,
                          e.cpu_total, e.optimizer_grad_share)


def max_model_size(plan: ParallelPlan, gpu_budget_bytes: float, base_params: float,
                   params_per_expert: float):
    """parallel.cpp:82-115 -> (max_experts, total_params)."""
    c = plan.to_c()
    n = C.c_int64()
    tot = C.c_double()
    _raise(L.load().moe_max_model_size(C.byref(c), float(gpu_budget_bytes), float(base_params),
                                       float(params_per_expert), C.byref(n), C.byref(tot)))
    return n.value, tot.value


def workspace_bytes(handle) -> int:
    v = C.c_size_t()
    st = L.load().moe_workspace_bytes(handle.h, C.byref(v))
    if st != L.MOE_OK:
        raise ShapeError("moe_workspace_bytes: bad handle")
    return int(v.value)


def layer_params(d_model: int, d_ff: int, num_experts: int):
    """(non-expert, expert) parameter counts of one MoE layer: gate [d,E];
    experts W1 [d,f] + b1 [f] + W2 [f,d] + b2 [d] (routing.hpp:120-128)."""
    return d_model * num_experts, num_experts * (2 * d_model * d_ff + d_ff + d_model)


def capacity_check(plan: ParallelPlan, nonexpert_params: float, expert_params: float, layers=(),
                   hbm_bytes: float | None = None, reserve: float = 0.05) -> dict:
    """Per-GPU bytes of the plan's parameter state (memory_per_gpu) plus the
    workspace every given MoeLayer/MoeHandle allocated, against HBM (the
    current device's total memory unless ``hbm_bytes``; ``reserve`` is kept
    free).  Raises ConfigError when it does not fit; returns the breakdown."""
    est = memory_per_gpu(plan, nonexpert_params, expert_params)
    ws = 0
    for lay in layers:
        ws += workspace_bytes(getattr(lay, "handle", lay))
    if hbm_bytes is None:
        import torch
        hbm_bytes = float(torch.cuda.get_device_properties(torch.cuda.current_device()).total_memory)
    need = est.gpu_total() + ws
    budget = hbm_bytes * (1.0 - reserve)
    out = dict(state_bytes=est.gpu_total(), workspace_bytes=ws, total_bytes=need, budget_bytes=budget,
               host_bytes=est.cpu_total())
    if need > budget:
        raise ConfigError(f"capacity check: {need / 2**30:.1f} GiB per GPU exceeds the "
                          f"{budget / 2**30:.1f} GiB budget")
    return out
