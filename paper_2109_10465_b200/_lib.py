"""ctypes binding of libmoe_b200.so (include/moe_b200.h).

The library is built in-tree (``python -m paper_2109_10465_b200.build`` or
``__graft_entry__.build()``).  There is no fallback: if the shared object is
missing or fails to load, importing the operators raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# MOE_B200_LIB: load a variant build instead (benchmarking scripts only)
LIB_PATH = os.environ.get("MOE_B200_LIB") or os.path.join(HERE, "libmoe_b200.so")

MOE_OK, MOE_SHAPE, MOE_CONFIG, MOE_NONFINITE, MOE_UNIFORM_SHAPE, MOE_INVALID_ARG = range(6)
MOE_CUDA, MOE_NCCL, MOE_UNSUPPORTED = 6, 7, 8
MOE_F32, MOE_BF16, MOE_F64 = 0, 1, 2


class moe_router_cfg(C.Structure):
    _fields_ = [
        ("num_experts", C.c_int),
        ("capacity_factor_train", C.c_double),
        ("capacity_factor_eval", C.c_double),
        ("jitter_eps", C.c_double),
        ("balance_coeff", C.c_double),
        ("assignment_mode", C.c_int),
        ("group_count", C.c_int),
        ("top_k", C.c_int),
        ("rng_seed", C.c_uint64),
    ]


class moe_parallel_plan(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("world_size", "expert_parallel", "model_parallel",
                                         "zero_stage", "offload")]


class moe_memory_estimate(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("nonexpert_params", "expert_params", "nonexpert_grads",
                                            "expert_grads", "nonexpert_optim", "expert_optim")] + \
        [("grad_optim_on_cpu", C.c_int)] + \
        [(n, C.c_double) for n in ("gpu_total", "cpu_total", "optimizer_grad_share")]


class moe_layer_dims(C.Structure):
    _fields_ = [
        ("max_tokens", C.c_int64),
        ("d_model", C.c_int64),
        ("d_ff", C.c_int64),
        ("dtype", C.c_int),
        ("ep_size", C.c_int),
        ("ep_rank", C.c_int),
    ]


VP = C.c_void_p
H = C.c_void_p  # moe_handle*

# name: (restype, argtypes)
_SIGS = {
    "moe_abi_version": (C.c_int, []),
    "moe_router_cfg_default": (None, [C.POINTER(moe_router_cfg)]),
    "moe_router_cfg_validate": (C.c_int, [C.POINTER(moe_router_cfg)]),
    "moe_capacity": (C.c_int, [C.c_int64, C.POINTER(moe_router_cfg), C.c_int, C.POINTER(C.c_int)]),
    "moe_create": (C.c_int, [C.POINTER(moe_router_cfg), C.POINTER(moe_layer_dims), C.POINTER(H)]),
    "moe_destroy": (C.c_int, [H]),
    "moe_last_error": (C.c_char_p, [H]),
    "moe_set_stream": (C.c_int, [H, VP]),
    "moe_check": (C.c_int, [H, C.POINTER(C.c_uint32)]),
    "moe_forward": (C.c_int, [H, C.c_int64, VP, VP, VP, VP, VP, VP, C.c_int, C.c_uint64, VP, VP, VP,
                              VP, VP, VP]),
    "moe_backward": (C.c_int, [H, VP, C.c_float, VP, VP, VP, VP, VP, VP, VP]),
    "moe_backward_ex": (C.c_int, [H, VP, C.c_float, VP, VP, VP, VP, VP, VP, VP, C.c_uint]),
    "moe_last_decision_stats": (C.c_int, [H, C.POINTER(C.c_int), C.POINTER(C.c_int64), VP]),
    "moe_gate": (C.c_int, [H, C.c_int64, VP, VP, C.c_int, C.c_uint64, VP, VP, VP]),
    "moe_assign": (C.c_int, [H, C.c_int64, VP, C.c_int, C.c_uint64, VP, C.POINTER(C.c_int)]),
    "moe_assign_mode": (C.c_int, [H, C.c_int64, VP, C.c_int, C.c_int, C.c_int, C.c_uint64, VP,
                                  C.POINTER(C.c_int)]),
    "moe_dispatch": (C.c_int, [H, C.c_int64, VP, VP, VP, C.c_int, VP, VP]),
    "moe_combine": (C.c_int, [H, C.c_int64, VP, VP, VP, C.c_int, VP, VP, VP]),
    "moe_balance_loss": (C.c_int, [H, C.c_int64, VP, VP, C.c_double, VP]),
    "moe_ep_unique_id_size": (C.c_size_t, []),
    "moe_ep_get_unique_id": (C.c_int, [VP]),
    "moe_ep_init": (C.c_int, [H, VP]),
    "moe_ep_traffic": (C.c_int, [H, VP, C.POINTER(C.c_double)]),
    "moe_ep_blob_size": (C.c_size_t, []),
    "moe_gemm_path": (C.c_int, [H, C.POINTER(C.c_int)]),
    "moe_forward_f64": (C.c_int, [H, C.c_int64, VP, VP, VP, VP, VP, VP, C.c_int, C.c_uint64, VP, VP, VP,
                                  VP, VP, VP]),
    "moe_backward_f64": (C.c_int, [H, VP, C.c_double, VP, VP, VP, VP, VP, VP, VP, C.c_int]),
    "moe_workspace_bytes": (C.c_int, [H, C.POINTER(C.c_size_t)]),
    "moe_plan_validate": (C.c_int, [C.POINTER(moe_parallel_plan)]),
    "moe_plan_last_error": (C.c_char_p, []),
    "moe_memory_per_gpu": (C.c_int, [C.POINTER(moe_parallel_plan), C.c_double, C.c_double,
                                     C.POINTER(moe_memory_estimate)]),
    "moe_max_model_size": (C.c_int, [C.POINTER(moe_parallel_plan), C.c_double, C.c_double, C.c_double,
                                     C.POINTER(C.c_int64), C.POINTER(C.c_double)]),
    "moe_ep_export": (C.c_int, [H, VP]),
    "moe_ep_import": (C.c_int, [H, VP]),
    "moe_profile_enable": (C.c_int, [H, C.c_int]),
    "moe_profile_read": (C.c_int, [H, C.c_int, C.c_char_p, C.POINTER(C.c_double),
                                   C.POINTER(C.c_int64), C.POINTER(C.c_int)]),
    "moe_kernel_launch_count": (C.c_uint64, []),
    "moe_debug_set_tensor_cores": (None, [C.c_int]),
    "moe_debug_mt64_chunk_host": (C.c_int, [C.c_uint64, C.c_int64, C.c_int, C.c_int64, VP]),
    "moe_debug_mt64_device": (C.c_int, [C.c_uint64, C.c_int64, VP]),
    "moe_accumulate_decision_stats": (C.c_int, [VP, VP, VP]),
    "moe_prefetch_jitter": (C.c_int, [VP, C.c_uint64, C.c_int64]),
    "moe_rng_permutation": (C.c_int, [C.c_uint64, C.c_int64, VP]),
    "moe_convert_f64": (C.c_int, [VP, C.c_int64, C.c_int, VP, VP]),
    "moe_grad_sqnorm": (C.c_int, [VP, C.c_int64, C.c_int, VP, VP]),
    "moe_clip_scale": (C.c_int, [VP, C.c_double, VP, VP]),
    "moe_adam_update": (C.c_int, [VP, VP, VP, VP, C.c_int64, C.c_int, VP, VP, C.c_double, C.c_double,
                                  C.c_double, C.c_double, C.c_int64, VP]),
    "moe_debug_jitter_device": (C.c_int, [C.c_uint64, C.c_int64, C.c_double, VP]),
    "moe_debug_rts_order": (C.c_int, [C.c_uint64, C.c_int64, VP]),
    "moe_debug_gate_stamps": (C.c_int, [VP, C.c_int, C.POINTER(C.c_int)]),
    "moe_debug_gate_tc_logits": (C.c_int, [VP, VP, VP, VP, C.c_int64, C.c_int, C.c_int, C.c_int]),
    "moe_debug_gate_tc_dw": (C.c_int, [VP, VP, VP, VP, C.c_int64, C.c_int, C.c_int, C.c_int]),
    "moe_debug_gate_tc_dx": (C.c_int, [C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, VP, VP, VP, VP,
                                       VP, VP, VP, C.c_int, VP, VP]),
    "moe_derive_seed_tag": (C.c_uint64, [C.c_uint64, C.c_char_p]),
    "moe_derive_seed_u64": (C.c_uint64, [C.c_uint64, C.c_uint64]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load() -> C.CDLL:
    """Load libmoe_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with "
                              "`python -m paper_2109_10465_b200.build` (no CPU fallback exists)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
