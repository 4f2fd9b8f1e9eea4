"""Python mirror of the reference's MoE-layer operator API
(/root/reference/proj/core/include/moeforge/routing.hpp), running on the
B200 kernels of libmoe_b200.so through the C ABI.

Names, argument meaning and error behaviour follow the reference:

=================================  =====================================
reference (routing.hpp)            here
=================================  =====================================
``Phase`` / ``AssignmentMode``     ``Phase`` / ``AssignmentMode``
``RouterConfig`` (+validate)       ``RouterConfig``
``kDropped``                       ``KDROPPED``
``RoutingDecision``                ``RoutingDecision`` (device tensors)
``capacity``                       ``capacity``
``gate_forward``/``GateResult``    ``gate_forward`` / ``GateResult``
``assign_plain/grouped/rts``       same names
``make_assignment``                ``make_assignment``
``dispatch``/``DispatchBuffer``    ``dispatch`` / ``DispatchBuffer``
``combine``                        ``combine``
``balance_loss``                   ``balance_loss``
``ExpertFfn``/``MoeLayerParams``   same (packed [E,...] tensors inside)
``moe_layer_forward``              ``moe_layer_forward`` (autograd-aware)
ShapeError/ConfigError/...         same exception names
=================================  =====================================

Tensors are torch CUDA tensors (device memory and streams only; every
computation is a kernel of libmoe_b200.so).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum

import torch

from . import _lib as L


# --- exceptions (common.hpp:10-35) -------------------------------------------
class MoeError(RuntimeError):
    pass


class ShapeError(MoeError, ValueError):
    pass


class NonFiniteError(MoeError):
    pass


class ConfigError(MoeError, ValueError):
    pass


class UniformShapeError(MoeError):
    pass


class InvalidArgument(MoeError, ValueError):
    pass


class CudaError(MoeError):
    pass


class NcclError(MoeError):
    pass


_EXC = {L.MOE_SHAPE: ShapeError, L.MOE_CONFIG: ConfigError, L.MOE_NONFINITE: NonFiniteError,
        L.MOE_UNIFORM_SHAPE: UniformShapeError, L.MOE_INVALID_ARG: InvalidArgument,
        L.MOE_CUDA: CudaError, L.MOE_NCCL: NcclError, L.MOE_UNSUPPORTED: MoeError}


def _check(status: int, handle=None, what: str = "") -> None:
    if status == L.MOE_OK:
        return
    msg = what
    if handle is not None:
        m = L.load().moe_last_error(handle)
        if m:
            msg = m.decode()
    raise _EXC.get(status, MoeError)(msg or f"moe status {status}")


class Phase(IntEnum):  # routing.hpp:13
    TRAIN = 0
    EVAL = 1


class AssignmentMode(IntEnum):  # routing.hpp:15
    PLAIN = 0
    GROUPED = 1
    RTS = 2


KDROPPED = -1  # routing.hpp:34


@dataclass
class RouterConfig:  # routing.hpp:17-32
    num_experts: int = 8
    capacity_factor_train: float = 1.0
    capacity_factor_eval: float = 2.0
    jitter_eps: float = 0.01
    balance_coeff: float = 0.01
    assignment_mode: AssignmentMode = AssignmentMode.PLAIN
    group_count: int = 1
    top_k: int = 1
    rng_seed: int = 0

    def to_c(self) -> L.moe_router_cfg:
        return L.moe_router_cfg(self.num_experts, self.capacity_factor_train,
                                self.capacity_factor_eval, self.jitter_eps, self.balance_coeff,
                                int(self.assignment_mode), self.group_count, self.top_k,
                                self.rng_seed)

    def validate(self) -> None:
        c = self.to_c()
        _check(L.load().moe_router_cfg_validate(C.byref(c)), what="router: invalid config")

    def capacity_factor(self, phase: Phase) -> float:
        return self.capacity_factor_train if phase == Phase.TRAIN else self.capacity_factor_eval

    def key(self):
        return (self.num_experts, self.capacity_factor_train, self.capacity_factor_eval,
                self.jitter_eps, self.balance_coeff, int(self.assignment_mode), self.group_count,
                self.top_k)


def derive_seed(seed: int, tag) -> int:
    """Rng::derive_seed (rng.cpp:24-34)."""
    lib = L.load()
    if isinstance(tag, str):
        return int(lib.moe_derive_seed_tag(seed, tag.encode()))
    return int(lib.moe_derive_seed_u64(seed, int(tag)))


def capacity(tokens: int, cfg: RouterConfig, phase: Phase) -> int:
    """routing.cpp:43-49: max(1, ceil(C_phase * tokens / E)); independent of top_k."""
    c = cfg.to_c()
    out = C.c_int()
    _check(L.load().moe_capacity(int(tokens), C.byref(c), int(phase), C.byref(out)),
           what="capacity: token count must be >= 1" if tokens < 1 else "router: invalid config")
    return out.value


def _dtype_code(t: torch.dtype) -> int:
    if t == torch.float32:
        return L.MOE_F32
    if t == torch.bfloat16:
        return L.MOE_BF16
    if t == torch.float64:
        return L.MOE_F64
    raise ConfigError(f"unsupported activation dtype {t}")


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _dense(t: torch.Tensor, device, name: str) -> None:
    """The kernels read raw row-major device memory: reject views and tensors
    on another device instead of reading them wrongly."""
    if not t.is_cuda or t.device != torch.device(device):
        raise ShapeError(f"moe_layer_forward: {name} must be on {device}")
    if not t.is_contiguous():
        raise ShapeError(f"moe_layer_forward: {name} must be contiguous")


# --- handles -------------------------------------------------------------------
class MoeHandle:
    """One moe_handle: workspace + saved forward context + stream binding."""

    def __init__(self, cfg: RouterConfig, max_tokens: int, d_model: int, d_ff: int,
                 dtype: torch.dtype, ep_size: int = 1, ep_rank: int = 0):
        lib = L.load()
        self.cfg = cfg
        self.dims = (max_tokens, d_model, d_ff, dtype, ep_size, ep_rank)
        c = cfg.to_c()
        dims = L.moe_layer_dims(max_tokens, d_model, d_ff, _dtype_code(dtype), ep_size, ep_rank)
        h = C.c_void_p()
        st = lib.moe_create(C.byref(c), C.byref(dims), C.byref(h))
        _check(st, None, "moe_create failed")
        self.h = h
        self.dtype = dtype
        self.max_tokens = max_tokens
        self.d_model, self.d_ff = d_model, d_ff
        self.ep_size, self.ep_rank = ep_size, ep_rank

    def __del__(self):
        try:
            if getattr(self, "h", None):
                L.load().moe_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def bind_stream(self):
        _check(L.load().moe_set_stream(self.h, C.c_void_p(torch.cuda.current_stream().cuda_stream)),
               self.h)

    def check(self) -> int:
        fl = C.c_uint32()
        _check(L.load().moe_check(self.h, C.byref(fl)), self.h)
        return fl.value

    def ep_init(self, unique_id: bytes):
        buf = C.create_string_buffer(unique_id, len(unique_id))
        _check(L.load().moe_ep_init(self.h, buf), self.h)

    def ep_bootstrap(self, all_gather, barrier):
        """NCCL-free binding of the NVLink peer map (moe_ep_export/import):
        ``all_gather(bytes) -> list[bytes]`` returns every rank's blob in rank
        order, ``barrier()`` synchronises the ranks (e.g. torch.distributed
        over gloo).  Ranks may share a GPU."""
        lib = L.load()
        n = lib.moe_ep_blob_size()
        mine = C.create_string_buffer(n)
        _check(lib.moe_ep_export(self.h, mine), self.h)
        blobs = all_gather(mine.raw)
        if len(blobs) != self.dims[4] or any(len(b) != n for b in blobs):
            raise ConfigError("ep_bootstrap: one blob per rank required")
        allb = C.create_string_buffer(b"".join(blobs), n * len(blobs))
        _check(lib.moe_ep_import(self.h, allb), self.h)
        barrier()

    def gemm_path(self) -> str:
        """'tcgen05' or 'simt': the kernel family of this handle's expert GEMMs."""
        v = C.c_int()
        _check(L.load().moe_gemm_path(self.h, C.byref(v)), self.h)
        return "tcgen05" if v.value == 1 else "simt"

    def profile(self, on: bool):
        """Enable the per-stage CUDA-event timeline (resets accumulators)."""
        _check(L.load().moe_profile_enable(self.h, 1 if on else 0), self.h)

    def profile_read(self) -> dict:
        """{stage: (total_ms, calls)} accumulated since profile(True)."""
        n = 64
        names = C.create_string_buffer(32 * n)
        ms = (C.c_double * n)()
        calls = (C.c_int64 * n)()
        cnt = C.c_int()
        _check(L.load().moe_profile_read(self.h, n, names, ms, calls, C.byref(cnt)), self.h)
        raw = names.raw
        return {raw[32 * i:32 * i + 32].split(b"\0")[0].decode(): (ms[i], calls[i])
                for i in range(cnt.value)}

    def stats(self):
        cap = C.c_int()
        drops = C.c_int64()
        kept = torch.empty(self.cfg.num_experts, dtype=torch.int64)
        _check(L.load().moe_last_decision_stats(self.h, C.byref(cap), C.byref(drops),
                                                C.c_void_p(kept.data_ptr())), self.h)
        return cap.value, drops.value, kept


def kernel_launch_count() -> int:
    """Kernels launched by libmoe_b200.so in this process so far."""
    return int(L.load().moe_kernel_launch_count())


def ep_unique_id() -> bytes:
    lib = L.load()
    n = lib.moe_ep_unique_id_size()
    buf = C.create_string_buffer(n)
    _check(lib.moe_ep_get_unique_id(buf), None, "ncclGetUniqueId failed")
    return buf.raw


_handle_cache: dict = {}


def _scratch_handle(cfg: RouterConfig, T: int, d: int, dtype: torch.dtype, f: int = 1,
                    min_cap: int = 0) -> MoeHandle:
    """A cached handle for the per-stage operators, large enough for T tokens
    and (assignment) an explicit capacity of min_cap."""
    key = (cfg.key(), d, f, dtype)
    h = _handle_cache.get(key)
    if h is None or h.max_tokens < T or getattr(h, "cap_ok", 0) < min_cap:
        T_alloc = max(T, 1, h.max_tokens if h is not None else 1)
        need = max(min_cap, getattr(h, "cap_ok", 0) if h is not None else 0)
        c = RouterConfig(**{**cfg.__dict__})
        c.capacity_factor_eval = max(c.capacity_factor_eval, need * c.num_experts / T_alloc + 1.0)
        h = MoeHandle(c, T_alloc, d, f, dtype)
        h.cap_ok = capacity(T_alloc, c, Phase.EVAL)
        _handle_cache[key] = h
    h.bind_stream()
    return h


# --- per-stage operators (routing.hpp:60-118) ------------------------------------
@dataclass
class RoutingDecision:  # routing.hpp:38-57
    num_experts: int
    capacity: int
    top_k: int
    expert_id: torch.Tensor  # int32 [T*k]
    slot: torch.Tensor       # int32 [T*k]
    gate_prob: torch.Tensor  # float32 [T*k]

    def tokens(self) -> int:
        return self.expert_id.numel() // self.top_k

    def kept(self, token: int, k: int = 0) -> bool:
        return int(self.slot[token * self.top_k + k]) != KDROPPED

    def drop_count(self) -> int:
        return int((self.slot == KDROPPED).sum())

    def kept_per_expert(self) -> torch.Tensor:
        m = self.slot != KDROPPED
        return torch.bincount(self.expert_id[m].long(), minlength=self.num_experts)


@dataclass
class GateResult:  # routing.hpp:62-66
    probs: torch.Tensor          # [T, E] fp32
    choice: torch.Tensor         # int32 [T*k]
    gate_prob: list              # per k: [T] fp32


def gate_forward(x: torch.Tensor, gate_w: torch.Tensor, cfg: RouterConfig, phase: Phase,
                 jitter_seed: int) -> GateResult:
    cfg.validate()
    if x.dim() != 2 or gate_w.dim() != 2 or x.shape[1] != gate_w.shape[0] or \
            gate_w.shape[1] != cfg.num_experts:
        raise ShapeError("gate_forward: x [T,d] and gate_w [d,E] required")
    T, d = x.shape
    E, K = cfg.num_experts, cfg.top_k
    h = _scratch_handle(cfg, T, d, x.dtype)
    x = x.contiguous()
    gw = gate_w.float().contiguous()
    probs = torch.empty(T, E, device=x.device, dtype=torch.float32)
    choice = torch.empty(T * K, device=x.device, dtype=torch.int32)
    gp = torch.empty(T * K, device=x.device, dtype=torch.float32)
    _check(L.load().moe_gate(h.h, T, _p(x), _p(gw), int(phase), jitter_seed, _p(probs),
                             _p(choice), _p(gp)), h.h)
    h.check()
    return GateResult(probs, choice, [gp.view(T, K)[:, k].contiguous() for k in range(K)])


def _assign(choice: torch.Tensor, num_experts: int, cap: int, top_k: int, mode: int,
            group_count: int, seed: int) -> RoutingDecision:
    choice = choice.to(torch.int32).contiguous()
    T = choice.numel() // top_k
    cfg = RouterConfig(num_experts=num_experts, top_k=top_k, group_count=max(group_count, 1))
    h = _scratch_handle(cfg, max(T, 1), 8, torch.float32, min_cap=cap)
    slot = torch.empty_like(choice)
    cap_out = C.c_int()
    _check(L.load().moe_assign_mode(h.h, T, _p(choice), cap, mode, group_count, seed, _p(slot),
                                    C.byref(cap_out)), h.h)
    return RoutingDecision(num_experts, cap_out.value, top_k, choice.clone(), slot,
                           torch.zeros(choice.numel(), device=choice.device))


def assign_plain(choice, num_experts: int, cap: int, top_k: int = 1) -> RoutingDecision:
    return _assign(choice, num_experts, cap, top_k, AssignmentMode.PLAIN, 1, 0)


def assign_grouped(choice, num_experts: int, cap: int, group_count: int,
                   top_k: int = 1) -> RoutingDecision:
    return _assign(choice, num_experts, cap, top_k, AssignmentMode.GROUPED, group_count, 0)


def assign_rts(choice, num_experts: int, cap: int, rng_seed: int,
               top_k: int = 1) -> RoutingDecision:
    return _assign(choice, num_experts, cap, top_k, AssignmentMode.RTS, 1, rng_seed)


def make_assignment(choice, tokens: int, cfg: RouterConfig, phase: Phase,
                    rng_seed: int) -> RoutingDecision:
    cap = capacity(tokens, cfg, phase)
    if phase == Phase.EVAL:  # routing.cpp:194-196
        return assign_plain(choice, cfg.num_experts, cap, cfg.top_k)
    if cfg.assignment_mode == AssignmentMode.PLAIN:
        return assign_plain(choice, cfg.num_experts, cap, cfg.top_k)
    if cfg.assignment_mode == AssignmentMode.GROUPED:
        return assign_grouped(choice, cfg.num_experts, cap, cfg.group_count, cfg.top_k)
    return assign_rts(choice, cfg.num_experts, cap, rng_seed, cfg.top_k)


@dataclass
class DispatchBuffer:  # routing.hpp:96-104
    data: torch.Tensor       # [E*capacity, d]
    num_experts: int
    capacity: int
    occupancy: torch.Tensor  # uint8 [E*capacity]


def dispatch(x: torch.Tensor, decision: RoutingDecision) -> DispatchBuffer:
    if x.dim() != 2 or x.shape[0] != decision.tokens():
        raise ShapeError("dispatch: x rows must match decision tokens")
    T, d = x.shape
    cfg = RouterConfig(num_experts=decision.num_experts, top_k=decision.top_k)
    h = _scratch_handle(cfg, T, d, x.dtype)
    rows = decision.num_experts * decision.capacity
    buf = torch.empty(rows, d, device=x.device, dtype=x.dtype)
    occ = torch.empty(rows, device=x.device, dtype=torch.uint8)
    _check(L.load().moe_dispatch(h.h, T, _p(x.contiguous()), _p(decision.expert_id),
                                 _p(decision.slot), decision.capacity, _p(buf), _p(occ)), h.h)
    return DispatchBuffer(buf, decision.num_experts, decision.capacity, occ)


def combine(expert_out: torch.Tensor, decision: RoutingDecision, residual: torch.Tensor,
            weights: list) -> torch.Tensor:
    T = decision.tokens()
    rows = decision.num_experts * decision.capacity
    if expert_out.dim() != 2 or expert_out.shape[0] != rows:
        raise ShapeError("combine: expert_out must be [E*capacity, d]")
    d = expert_out.shape[1]
    if residual.dim() != 2 or residual.shape[0] != T or residual.shape[1] != d:
        raise ShapeError("combine: residual must be [T, d]")
    if len(weights) != decision.top_k:
        raise ShapeError("combine: one weight tensor per route required")
    for w in weights:
        if w.numel() != T:
            raise ShapeError("combine: weight tensor must have one entry per token")
    cfg = RouterConfig(num_experts=decision.num_experts, top_k=decision.top_k)
    h = _scratch_handle(cfg, T, d, expert_out.dtype)
    wts = torch.stack([w.reshape(-1).float() for w in weights]).contiguous()
    y = torch.empty(T, d, device=expert_out.device, dtype=expert_out.dtype)
    _check(L.load().moe_combine(h.h, T, _p(expert_out.contiguous()), _p(decision.expert_id),
                                _p(decision.slot), decision.capacity,
                                _p(residual.to(expert_out.dtype).contiguous()), _p(wts), _p(y)), h.h)
    return y


def balance_loss(probs: torch.Tensor, decision: RoutingDecision, alpha: float) -> torch.Tensor:
    if probs.dim() != 2 or probs.shape[0] != decision.tokens() or \
            probs.shape[1] != decision.num_experts:
        raise ShapeError("balance_loss: probs must be [T, E]")
    T, E = probs.shape
    cfg = RouterConfig(num_experts=E, top_k=decision.top_k)
    h = _scratch_handle(cfg, T, 8, torch.float32)
    out = torch.empty(1, device=probs.device, dtype=torch.float32)
    _check(L.load().moe_balance_loss(h.h, T, _p(probs.float().contiguous()),
                                     _p(decision.expert_id), alpha, _p(out)), h.h)
    return out[0]


# --- full layer ------------------------------------------------------------------
@dataclass
class ExpertFfn:  # routing.hpp:120-123
    w1: torch.Tensor  # [d, f]
    b1: torch.Tensor  # [f]
    w2: torch.Tensor  # [f, d]
    b2: torch.Tensor  # [d]


@dataclass
class MoeLayerParams:  # routing.hpp:125-128, packed on device as [E, ...]
    gate_w: torch.Tensor          # [d, E] fp32
    w1: torch.Tensor              # [E, d, f]
    b1: torch.Tensor              # [E, f] fp32
    w2: torch.Tensor              # [E, f, d]
    b2: torch.Tensor              # [E, d] fp32

    @staticmethod
    def from_experts(gate_w: torch.Tensor, experts: list, dtype=None) -> "MoeLayerParams":
        dt = dtype or experts[0].w1.dtype
        return MoeLayerParams(gate_w.float().contiguous(),
                              torch.stack([e.w1 for e in experts]).to(dt).contiguous(),
                              torch.stack([e.b1 for e in experts]).float().contiguous(),
                              torch.stack([e.w2 for e in experts]).to(dt).contiguous(),
                              torch.stack([e.b2 for e in experts]).float().contiguous())

    @property
    def experts(self) -> list:
        return [ExpertFfn(self.w1[e], self.b1[e], self.w2[e], self.b2[e])
                for e in range(self.w1.shape[0])]


@dataclass
class MoeLayerResult:  # routing.hpp:130-134
    y: torch.Tensor
    aux_loss: torch.Tensor
    decision: RoutingDecision


class MoeLayer:
    """A B200 MoE layer bound to one handle (workspace + saved context).

    ``forward`` / ``backward`` are the raw C-ABI calls; ``__call__`` is the
    autograd-aware form (the tape adapter of SURVEY §8b)."""

    def __init__(self, cfg: RouterConfig, max_tokens: int, d_model: int, d_ff: int,
                 dtype: torch.dtype = torch.bfloat16, ep_size: int = 1, ep_rank: int = 0):
        cfg.validate()
        self.cfg = cfg
        self.handle = MoeHandle(cfg, max_tokens, d_model, d_ff, dtype, ep_size, ep_rank)
        self.dtype = dtype
        self.d_model, self.d_ff = d_model, d_ff
        self.ep_size, self.ep_rank = ep_size, ep_rank
        self.n_local = cfg.num_experts // ep_size
        # forward generation: the handle keeps ONE saved context, so an
        # autograd node may only run backward for the latest forward
        self._gen = 0

    def _check_params(self, p: MoeLayerParams, device):
        E, El, d, f = self.cfg.num_experts, self.n_local, self.d_model, self.d_ff
        if tuple(p.gate_w.shape) != (d, E) or tuple(p.w1.shape) != (El, d, f) or \
                tuple(p.w2.shape) != (El, f, d) or tuple(p.b1.shape) != (El, f) or \
                tuple(p.b2.shape) != (El, d):
            raise ShapeError("moe_layer_forward: expert count does not match config")
        if p.w1.dtype != self.dtype or p.w2.dtype != self.dtype:
            raise ShapeError("moe_layer_forward: expert weight dtype does not match the layer")
        side = torch.float64 if self.dtype == torch.float64 else torch.float32
        for name in ("gate_w", "b1", "b2"):
            if getattr(p, name).dtype != side:
                raise ShapeError(f"moe_layer_forward: {name} must be {side}")
        for name in ("gate_w", "w1", "b1", "w2", "b2"):
            _dense(getattr(p, name), device, name)

    def forward(self, x, params: MoeLayerParams, phase: Phase, seed: int, residual=None,
                y=None, aux=None, decision: bool = True, check: bool = True):
        if x.dim() != 2 or x.shape[1] != self.d_model or x.dtype != self.dtype:
            raise ShapeError("moe_layer_forward: x must be [T, d_model] of the layer dtype")
        _dense(x, x.device, "x")
        self._check_params(params, x.device)
        if residual is not None:
            if tuple(residual.shape) != tuple(x.shape) or residual.dtype != self.dtype:
                raise ShapeError("moe_layer_forward: residual must be [T, d_model] of the layer dtype")
            _dense(residual, x.device, "residual")
        for name, t in (("y", y), ("aux", aux)):
            if t is not None:
                _dense(t, x.device, name)
        T = x.shape[0]
        K = self.cfg.top_k
        dev = x.device
        self.handle.bind_stream()
        f64 = self.dtype == torch.float64
        side = torch.float64 if f64 else torch.float32
        y = torch.empty_like(x) if y is None else y
        aux = torch.empty(1, device=dev, dtype=side) if aux is None else aux
        eid = slot = gp = None
        if decision:
            eid = torch.empty(T * K, device=dev, dtype=torch.int32)
            slot = torch.empty(T * K, device=dev, dtype=torch.int32)
            gp = torch.empty(T * K, device=dev, dtype=side)
        fwd = L.load().moe_forward_f64 if f64 else L.load().moe_forward
        _check(fwd(self.handle.h, T, _p(x), _p(params.gate_w), _p(params.w1), _p(params.b1), _p(params.w2),
                   _p(params.b2), int(phase), seed, _p(residual), _p(y), _p(aux), _p(eid), _p(slot), _p(gp)),
               self.handle.h)
        if check:
            self.handle.check()
        dec = None
        if decision:
            cap = capacity(T, self.cfg, phase)
            if self.cfg.assignment_mode == AssignmentMode.GROUPED and phase == Phase.TRAIN:
                G = self.cfg.group_count
                cap = G * ((cap + G - 1) // G)
            dec = RoutingDecision(self.cfg.num_experts, cap, K, eid, slot, gp)
        # keep every tensor the saved context points at alive until backward
        # (the reference tape keeps its parents alive the same way, tensor.cpp:140-152)
        self._saved = (params, residual is not None, x, residual)
        self._gen += 1
        return y, aux, dec

    def backward(self, dy, daux: float = 1.0, check: bool = True, grads=None, accumulate: bool = False,
                 weights_f32: bool = False):
        """Backward of <dy, y> + daux * aux for the last forward (moe_backward_ex).
        ``accumulate``: add into ``grads`` instead of writing them (the tape's
        +=); ``weights_f32``: dw1 / dw2 of a bf16 layer in float32 (fp32
        masters).  ``grads`` is allocated when None."""
        params, has_res, x = self._saved[:3]
        if tuple(dy.shape) != tuple(x.shape) or dy.dtype != self.dtype:
            raise ShapeError("moe_layer_backward: dy must be [T, d_model] of the layer dtype")
        El, d, f = self.n_local, self.d_model, self.d_ff
        dev = dy.device
        f64 = self.dtype == torch.float64
        side = torch.float64 if f64 else torch.float32
        wdt = torch.float32 if (weights_f32 and self.dtype == torch.bfloat16) else self.dtype
        if grads is None:
            grads = dict(dx=torch.empty_like(dy),
                         dgate_w=torch.empty_like(params.gate_w),
                         dw1=torch.empty(El, d, f, device=dev, dtype=wdt),
                         db1=torch.empty(El, f, device=dev, dtype=side),
                         dw2=torch.empty(El, f, d, device=dev, dtype=wdt),
                         db2=torch.empty(El, d, device=dev, dtype=side),
                         dresidual=torch.empty_like(dy) if has_res else None)
            accumulate = False
        g = grads
        self.handle.bind_stream()
        if f64:
            _check(L.load().moe_backward_f64(self.handle.h, _p(dy.contiguous()), float(daux), _p(g["dx"]),
                                             _p(g["dgate_w"]), _p(g["dw1"]), _p(g["db1"]), _p(g["dw2"]),
                                             _p(g["db2"]), _p(g.get("dresidual")), int(bool(accumulate))),
                   self.handle.h)
        else:
            flags = (1 if accumulate else 0) | (2 if weights_f32 else 0)
            _check(L.load().moe_backward_ex(self.handle.h, _p(dy.contiguous()), float(daux), _p(g["dx"]),
                                            _p(g["dgate_w"]), _p(g["dw1"]), _p(g["db1"]), _p(g["dw2"]),
                                            _p(g["db2"]), _p(g.get("dresidual")), flags), self.handle.h)
        if check:
            self.handle.check()
        return grads

    def __call__(self, x, params: MoeLayerParams, phase: Phase, seed: int, residual=None):
        return moe_layer_forward(x, params, self.cfg, phase, seed, residual, layer=self)

    def ep_init(self, unique_id: bytes):
        self.handle.ep_init(unique_id)

    def ep_bootstrap(self, all_gather, barrier):
        self.handle.ep_bootstrap(all_gather, barrier)

    def prefetch_jitter(self, seed: int, tokens: int):
        """moe_prefetch_jitter: generate the jitter stream of a later forward
        with this seed during the next forward/backward call, next to its
        expert GEMMs (values unchanged).  Call before forward(seed_i) with
        seed_{i+1}."""
        _check(L.load().moe_prefetch_jitter(self.handle.h, seed, tokens), self.handle.h)


class _MoeFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, layer, params, phase, seed, x, gate_w, w1, b1, w2, b2, residual):
        y, aux, dec = layer.forward(x, params, phase, seed, residual)
        ctx.layer = layer
        ctx.gen = layer._gen
        ctx.has_res = residual is not None
        layer._last_dec = dec
        return y, aux[0]

    @staticmethod
    def backward(ctx, dy, daux):
        if ctx.layer._gen != ctx.gen:
            raise MoeError("moe_layer_forward: this MoeLayer ran another forward before this "
                           "node's backward; its handle keeps only the latest forward context "
                           "(use one MoeLayer per in-flight forward)")
        daux_v = 0.0 if daux is None else float(daux)
        g = ctx.layer.backward(dy.to(ctx.layer.dtype).contiguous(), daux_v)
        return (None, None, None, None, g["dx"], g["dgate_w"], g["dw1"], g["db1"], g["dw2"],
                g["db2"], g["dresidual"] if ctx.has_res else None)


def moe_layer_forward(x: torch.Tensor, params: MoeLayerParams, cfg: RouterConfig, phase: Phase,
                      seed: int, residual: torch.Tensor | None = None,
                      layer: MoeLayer | None = None) -> MoeLayerResult:
    """routing.cpp:376-424 on the B200 kernels.  Autograd-aware: gradients of
    ``y`` and ``aux_loss`` flow into x, residual and every parameter."""
    cfg.validate()
    if params.w1.shape[0] != cfg.num_experts and (layer is None or layer.ep_size == 1):
        raise ShapeError("moe_layer_forward: expert count does not match config")
    T, d = x.shape
    f = params.w1.shape[-1]
    if layer is None:
        layer = MoeLayer(cfg, T, d, f, x.dtype)
    y, aux = _MoeFn.apply(layer, params, phase, seed, x, params.gate_w, params.w1, params.b1,
                          params.w2, params.b2, residual)
    return MoeLayerResult(y, aux, layer._last_dec)
