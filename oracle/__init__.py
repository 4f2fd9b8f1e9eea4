"""oracle — CPU parity checkers for the B200 MoE layer (TEST INFRASTRUCTURE ONLY).

Two interchangeable backends with identical signatures:

* ``restatement()`` — ``liboracle.so``, the plain-C restatement in
  ``moe_oracle.c`` of routing.cpp / rng.cpp / ops.cpp / parallel.cpp.
* ``reference()``   — ``_ref/libmoeforge_ref.so``, the reference itself compiled
  from its unmodified sources (``oracle/Makefile``), when it has been built.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu baseline and
``--impl reference``) may import this package.  The product package
``paper_2109_10465_b200`` never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
TRAIN, EVAL = 0, 1
PLAIN, GROUPED, RTS = 0, 1, 2
KDROPPED = -1


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: oracle status {status}")
        self.status = status


class Cfg(C.Structure):
    """RouterConfig (routing.hpp:17-32) in the layout of orc_cfg."""

    _fields_ = [
        ("num_experts", C.c_int),
        ("capacity_factor_train", C.c_double),
        ("capacity_factor_eval", C.c_double),
        ("jitter_eps", C.c_double),
        ("balance_coeff", C.c_double),
        ("assignment_mode", C.c_int),
        ("group_count", C.c_int),
        ("top_k", C.c_int),
    ]


def make_cfg(num_experts=8, capacity_factor_train=1.0, capacity_factor_eval=2.0, jitter_eps=0.01,
             balance_coeff=0.01, assignment_mode=PLAIN, group_count=1, top_k=1) -> Cfg:
    return Cfg(num_experts, capacity_factor_train, capacity_factor_eval, jitter_eps, balance_coeff,
               assignment_mode, group_count, top_k)


def build(ref: bool = False) -> None:
    targets = ["all"] + (["ref"] if ref else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _p(a, ct):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ct))


D = C.POINTER(C.c_double)
I32 = C.POINTER(C.c_int32)


@dataclass
class LayerOut:
    y: np.ndarray
    aux: float
    expert_id: np.ndarray
    slot: np.ndarray
    gate_prob: np.ndarray
    capacity: int
    dx: np.ndarray | None = None
    dgate_w: np.ndarray | None = None
    dw1: np.ndarray | None = None
    db1: np.ndarray | None = None
    dw2: np.ndarray | None = None
    db2: np.ndarray | None = None
    dresidual: np.ndarray | None = None


class _Backend:
    def __init__(self, path: str, prefix: str):
        self.path = path
        self.lib = C.CDLL(path)
        self.prefix = prefix
        L = self.lib
        f = lambda n: getattr(L, prefix + n)  # noqa: E731
        self._derive_tag = f("derive_seed_tag")
        self._derive_tag.restype = C.c_uint64
        self._derive_tag.argtypes = [C.c_uint64, C.c_char_p]
        self._derive_u64 = f("derive_seed_u64")
        self._derive_u64.restype = C.c_uint64
        self._derive_u64.argtypes = [C.c_uint64, C.c_uint64]
        self._mt = f("mt64_raw")
        self._mt.restype = None
        self._mt.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.POINTER(C.c_uint64)]
        self._perm = f("permutation")
        self._perm.argtypes = [C.c_uint64, C.c_int64, C.POINTER(C.c_uint32)]
        self._cap = f("capacity")
        self._cap.argtypes = [C.c_int64, C.POINTER(Cfg), C.c_int, C.POINTER(C.c_int)]
        self._assign = f("assign")
        self._assign.argtypes = [I32, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                 C.c_uint64, I32, C.POINTER(C.c_int)]
        self._layer = f("moe_layer")
        self._layer.argtypes = [D, D, D, D, D, D, C.c_int64, C.c_int64, C.c_int64, C.POINTER(Cfg),
                                C.c_int, C.c_uint64, D, D, D, I32, I32, D, C.POINTER(C.c_int), D,
                                C.c_double, D, D, D, D, D, D, D]
        self._ep = f("ep_forward")
        self._ep.argtypes = [D, C.c_int, C.c_int64, C.c_int64, C.c_int64, D, D, D, D, D,
                             C.POINTER(Cfg), C.c_int, C.c_uint64, D, I32, I32, D,
                             C.POINTER(C.c_int), D]

    # --- rng.cpp ---
    def derive_seed(self, seed: int, tag) -> int:
        if isinstance(tag, str):
            return int(self._derive_tag(seed, tag.encode()))
        return int(self._derive_u64(seed, tag))

    def mt64(self, seed: int, n: int, skip: int = 0) -> np.ndarray:
        out = np.empty(n, np.uint64)
        self._mt(seed, skip, n, _p(out, C.c_uint64))
        return out

    def permutation(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(max(n, 1), np.uint32)
        self._perm(seed, n, _p(out, C.c_uint32))
        return out[:n]

    # --- routing.cpp ---
    def capacity(self, tokens: int, cfg: Cfg, phase: int) -> int:
        c = C.c_int()
        st = self._cap(tokens, C.byref(cfg), phase, C.byref(c))
        if st:
            raise OracleError(st, "capacity")
        return c.value

    def assign(self, choice, num_experts, cap, top_k=1, mode=PLAIN, group_count=1, rts_seed=0):
        choice = np.ascontiguousarray(choice, np.int32)
        T = choice.size // top_k
        slot = np.empty(max(choice.size, 1), np.int32)
        capo = C.c_int()
        st = self._assign(_p(choice, C.c_int32), T, num_experts, cap, top_k, mode, group_count,
                          rts_seed, _p(slot, C.c_int32), C.byref(capo))
        if st:
            raise OracleError(st, "assign")
        return slot[: choice.size], capo.value

    def moe_layer(self, x, gate_w, w1, b1, w2, b2, cfg: Cfg, phase: int, seed: int,
                  residual=None, dy=None, daux: float = 1.0) -> LayerOut:
        x = np.ascontiguousarray(x, np.float64)
        T, d = x.shape
        E = cfg.num_experts
        f = w1.shape[-1]
        K = cfg.top_k
        arrs = [np.ascontiguousarray(a, np.float64) for a in (gate_w, w1, b1, w2, b2)]
        res = None if residual is None else np.ascontiguousarray(residual, np.float64)
        y = np.empty((T, d))
        aux = C.c_double()
        eid = np.empty(T * K, np.int32)
        slot = np.empty(T * K, np.int32)
        gp = np.empty(T * K)
        cap = C.c_int()
        grads = None
        if dy is not None:
            dy = np.ascontiguousarray(dy, np.float64)
            grads = [np.empty((T, d)), np.empty((d, E)), np.empty((E, d, f)), np.empty((E, f)),
                     np.empty((E, f, d)), np.empty((E, d)),
                     np.empty((T, d)) if res is not None else None]
        g = grads or [None] * 7
        st = self._layer(_p(x, C.c_double), *[_p(a, C.c_double) for a in arrs], T, d, f,
                         C.byref(cfg), phase, seed, _p(res, C.c_double), _p(y, C.c_double),
                         C.byref(aux), _p(eid, C.c_int32), _p(slot, C.c_int32),
                         _p(gp, C.c_double), C.byref(cap), _p(dy, C.c_double), daux,
                         *[_p(a, C.c_double) for a in g])
        if st:
            raise OracleError(st, "moe_layer")
        out = LayerOut(y, aux.value, eid, slot, gp, cap.value)
        if grads:
            (out.dx, out.dgate_w, out.dw1, out.db1, out.dw2, out.db2, out.dresidual) = grads
        return out

    def ep_forward(self, xs, gate_w, w1, b1, w2, b2, cfg: Cfg, phase: int, seed: int):
        xs = np.ascontiguousarray(xs, np.float64)
        ep, T, d = xs.shape
        f = w1.shape[-1]
        arrs = [np.ascontiguousarray(a, np.float64) for a in (gate_w, w1, b1, w2, b2)]
        ys = np.empty_like(xs)
        eid = np.empty(ep * T, np.int32)
        slot = np.empty(ep * T, np.int32)
        gp = np.empty(ep * T)
        cap = C.c_int()
        traffic = np.empty((ep, ep))
        st = self._ep(_p(xs, C.c_double), ep, T, d, f, *[_p(a, C.c_double) for a in arrs],
                      C.byref(cfg), phase, seed, _p(ys, C.c_double), _p(eid, C.c_int32),
                      _p(slot, C.c_int32), _p(gp, C.c_double), C.byref(cap),
                      _p(traffic, C.c_double))
        if st:
            raise OracleError(st, "ep_forward")
        return ys, eid.reshape(ep, T), slot.reshape(ep, T), gp.reshape(ep, T), cap.value, traffic


class _Restatement(_Backend):
    """Adds the per-stage entry points only the C restatement exports."""

    def __init__(self, path: str):
        super().__init__(path, "orc_")
        L = self.lib
        L.orc_gate_forward.argtypes = [D, D, C.c_int64, C.c_int64, C.POINTER(Cfg), C.c_int,
                                       C.c_uint64, D, I32, D, D]
        L.orc_dispatch.argtypes = [D, C.c_int64, C.c_int64, I32, I32, C.c_int, C.c_int, C.c_int,
                                   D, C.POINTER(C.c_uint8)]
        L.orc_combine.argtypes = [D, C.c_int64, C.c_int64, I32, I32, C.c_int, C.c_int, C.c_int,
                                  D, D, D]
        L.orc_balance_loss.argtypes = [D, C.c_int64, C.c_int, I32, C.c_int, C.c_double, D]

    def gate_forward(self, x, gate_w, cfg: Cfg, phase: int, jitter_seed: int):
        x = np.ascontiguousarray(x, np.float64)
        gw = np.ascontiguousarray(gate_w, np.float64)
        T, d = x.shape
        E, K = cfg.num_experts, cfg.top_k
        probs = np.empty((T, E))
        choice = np.empty(T * K, np.int32)
        gp = np.empty(T * K)
        noise = np.empty((T, d))
        st = self.lib.orc_gate_forward(_p(x, C.c_double), _p(gw, C.c_double), T, d, C.byref(cfg),
                                       phase, jitter_seed, _p(probs, C.c_double),
                                       _p(choice, C.c_int32), _p(gp, C.c_double),
                                       _p(noise, C.c_double))
        if st:
            raise OracleError(st, "gate_forward")
        return probs, choice, gp, noise

    def dispatch(self, x, expert_id, slot, top_k, num_experts, cap):
        x = np.ascontiguousarray(x, np.float64)
        T, d = x.shape
        eid = np.ascontiguousarray(expert_id, np.int32)
        sl = np.ascontiguousarray(slot, np.int32)
        buf = np.empty((num_experts * cap, d))
        occ = np.empty(num_experts * cap, np.uint8)
        st = self.lib.orc_dispatch(_p(x, C.c_double), T, d, _p(eid, C.c_int32), _p(sl, C.c_int32),
                                   top_k, num_experts, cap, _p(buf, C.c_double),
                                   _p(occ, C.c_uint8))
        if st:
            raise OracleError(st, "dispatch")
        return buf, occ

    def combine(self, expert_out, expert_id, slot, top_k, num_experts, cap, residual, weights):
        O_ = np.ascontiguousarray(expert_out, np.float64)
        res = np.ascontiguousarray(residual, np.float64)
        T, d = res.shape
        w = np.ascontiguousarray(weights, np.float64).reshape(top_k, T)
        eid = np.ascontiguousarray(expert_id, np.int32)
        sl = np.ascontiguousarray(slot, np.int32)
        y = np.empty((T, d))
        st = self.lib.orc_combine(_p(O_, C.c_double), T, d, _p(eid, C.c_int32), _p(sl, C.c_int32),
                                  top_k, num_experts, cap, _p(res, C.c_double), _p(w, C.c_double),
                                  _p(y, C.c_double))
        if st:
            raise OracleError(st, "combine")
        return y

    def balance_loss(self, probs, expert_id, top_k, alpha):
        P = np.ascontiguousarray(probs, np.float64)
        T, E = P.shape
        eid = np.ascontiguousarray(expert_id, np.int32)
        out = C.c_double()
        st = self.lib.orc_balance_loss(_p(P, C.c_double), T, E, _p(eid, C.c_int32), top_k, alpha,
                                       C.byref(out))
        if st:
            raise OracleError(st, "balance_loss")
        return out.value


_cache: dict[str, _Backend] = {}

REF_PATH = os.path.join(HERE, "_ref", "libmoeforge_ref.so")
ORC_PATH = os.path.join(HERE, "liboracle.so")


def restatement() -> _Restatement:
    if "orc" not in _cache:
        if not os.path.exists(ORC_PATH):
            build()
        _cache["orc"] = _Restatement(ORC_PATH)
    return _cache["orc"]


def have_reference() -> bool:
    return os.path.exists(REF_PATH)


def reference() -> _Backend:
    if "ref" not in _cache:
        _cache["ref"] = _Backend(REF_PATH, "ref_")
        lib = _cache["ref"].lib
        lib.ref_time_layer_mt.restype = C.c_double
        lib.ref_time_layer_mt.argtypes = [D, D, D, D, D, D, C.c_int64, C.c_int64, C.c_int64,
                                          C.POINTER(Cfg), C.c_int, C.c_uint64, D, C.c_int,
                                          C.POINTER(C.c_int)]
    return _cache["ref"]


def time_reference_layer(x, gate_w, w1, b1, w2, b2, cfg: Cfg, phase: int, seed: int, dy,
                         threads: int) -> float:
    """Wall seconds for `threads` concurrent reference fwd+bwd replicas."""
    ref = reference()
    arrs = [np.ascontiguousarray(a, np.float64) for a in (x, gate_w, w1, b1, w2, b2, dy)]
    T, d = arrs[0].shape
    f = arrs[2].shape[-1]
    st = C.c_int()
    secs = ref.lib.ref_time_layer_mt(*[_p(a, C.c_double) for a in arrs[:6]], T, d, f,
                                     C.byref(cfg), phase, seed, _p(arrs[6], C.c_double), threads,
                                     C.byref(st))
    if st.value:
        raise OracleError(st.value, "ref_time_layer_mt")
    return secs


# ---------------------------------------------------------------------------
# Synthetic inputs: drawn from the reference Rng streams so
# every backend sees identical values.
# ---------------------------------------------------------------------------
def uniform(seed: int, n: int, lo: float, hi: float) -> np.ndarray:
    """n draws of Rng::uniform(lo, hi) (rng.cpp:36-43) from Rng(seed)."""
    raw = restatement().mt64(seed, n)
    u = (raw >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return lo + (hi - lo) * u


def layer_inputs(T, d, f, E, seed=42, xscale=1.0, gscale=None, wscale=None, bscale=0.01):
    """x ~ U(-1,1); Wg, W1, W2 ~ U(-s,s) with s = sqrt(6/(fan_in+fan_out)); b ~ U(-.01,.01)."""
    o = restatement()
    gscale = gscale if gscale is not None else float(np.sqrt(6.0 / (d + E)))
    wscale = wscale if wscale is not None else float(np.sqrt(6.0 / (d + f)))
    x = uniform(o.derive_seed(seed, "x"), T * d, -xscale, xscale).reshape(T, d)
    gw = uniform(o.derive_seed(seed, "gate"), d * E, -gscale, gscale).reshape(d, E)
    w1 = uniform(o.derive_seed(seed, "w1"), E * d * f, -wscale, wscale).reshape(E, d, f)
    b1 = uniform(o.derive_seed(seed, "b1"), E * f, -bscale, bscale).reshape(E, f)
    w2 = uniform(o.derive_seed(seed, "w2"), E * f * d, -wscale, wscale).reshape(E, f, d)
    b2 = uniform(o.derive_seed(seed, "b2"), E * d, -bscale, bscale).reshape(E, d)
    dy = uniform(o.derive_seed(seed, "dy"), T * d, -1.0, 1.0).reshape(T, d)
    return x, gw, w1, b1, w2, b2, dy


# ---------------------------------------------------------------------------
# Expert optimizer step: AdamOptimizer, optim.cpp:10-57
# ---------------------------------------------------------------------------
def adam_restated(thetas, grads_per_step, lrs, clip=0.0, beta1=0.9, beta2=0.999, eps=1e-8):
    """f64 restatement of AdamOptimizer::step (optim.cpp:21-57) applied
    len(lrs) times.  thetas: list of flat arrays; grads_per_step[s][i] the
    gradient of tensor i at step s.  Returns (thetas, ms, vs)."""
    th = [np.array(t, np.float64, copy=True) for t in thetas]
    m = [np.zeros_like(t) for t in th]
    v = [np.zeros_like(t) for t in th]
    for s, lr in enumerate(lrs):
        if lr <= 0.0:
            raise ValueError("adam: learning rate must be positive")       # optim.cpp:22-24
        scale = 1.0
        if clip > 0.0:                                                      # optim.cpp:26-37
            sq = 0.0
            for g in grads_per_step[s]:
                for x in np.asarray(g, np.float64).ravel():                 # sequential order
                    sq += x * x
            norm = np.sqrt(sq)
            if norm > clip:
                scale = clip / norm
        step = s + 1                                                        # optim.cpp:38
        bc1 = 1.0 - beta1 ** step
        bc2 = 1.0 - beta2 ** step
        for i in range(len(th)):                                            # optim.cpp:41-55
            g = np.asarray(grads_per_step[s][i], np.float64) * scale
            m[i] = beta1 * m[i] + (1.0 - beta1) * g
            v[i] = beta2 * v[i] + (1.0 - beta2) * g * g
            th[i] = th[i] - lr * (m[i] / bc1) / (np.sqrt(v[i] / bc2) + eps)
    return th, m, v


def adam_reference(thetas, grads_per_step, lrs, clip=0.0, beta1=0.9, beta2=0.999, eps=1e-8):
    """The reference's own AdamOptimizer (oracle/_ref), same contract."""
    lib = reference().lib
    fn = lib.ref_adam
    fn.argtypes = [C.c_int, C.POINTER(C.c_int64), D, D, C.c_int, D, C.c_double, C.c_double,
                   C.c_double, C.c_double, D, D]
    n = len(thetas)
    numel = np.array([np.asarray(t).size for t in thetas], np.int64)
    th = np.ascontiguousarray(np.concatenate([np.asarray(t, np.float64).ravel() for t in thetas]))
    gs = np.ascontiguousarray(np.stack([np.concatenate([np.asarray(g, np.float64).ravel() for g in gl])
                                        for gl in grads_per_step]))
    lr = np.ascontiguousarray(np.asarray(lrs, np.float64))
    m = np.zeros_like(th)
    v = np.zeros_like(th)
    st = fn(n, numel.ctypes.data_as(C.POINTER(C.c_int64)), _p(th, C.c_double), _p(gs, C.c_double),
            len(lrs), _p(lr, C.c_double), clip, beta1, beta2, eps, _p(m, C.c_double), _p(v, C.c_double))
    if st:
        raise OracleError(st, "ref_adam")
    split = np.cumsum(numel)[:-1]
    return np.split(th, split), np.split(m, split), np.split(v, split)


# ---------------------------------------------------------------------------
# Checkpoints: written and pruned by the reference's
# own checkpoint.cpp / surgery.cpp (oracle/_ref) for the loader's parity tests.
# ---------------------------------------------------------------------------
def ref_save_toy_checkpoint(path, vocab=50, d_model=64, ffn_dim=128, enc_layers=2, dec_layers=2,
                            heads=2, num_experts=8, moe_every=2, seed=7):
    fn = reference().lib.ref_save_toy_checkpoint
    fn.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                   C.c_int, C.c_uint64]
    st = fn(str(path).encode(), vocab, d_model, ffn_dim, enc_layers, dec_layers, heads, num_experts,
            moe_every, seed)
    if st:
        raise OracleError(st, "ref_save_toy_checkpoint")


def ref_prune_checkpoint(src, dst, k, strategy="top_utilization", counts=None, seed=0):
    fn = reference().lib.ref_prune_checkpoint
    fn.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_int64), C.c_uint64]
    cp = None
    if counts is not None:
        arr = np.ascontiguousarray(np.asarray(counts, np.int64))
        cp = arr.ctypes.data_as(C.POINTER(C.c_int64))
    st = fn(str(src).encode(), str(dst).encode(), k, 0 if strategy == "top_utilization" else 1, cp, seed)
    if st:
        raise OracleError(st, "ref_prune_checkpoint")
