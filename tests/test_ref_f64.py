"""Pins tests/ref_f64.py (the f64 recomputation used for the full-size GPU
parity checks) to the C restatement: fed the restatement's own decisions, it
reproduces the restatement's y, aux and every gradient to ~1e-12 (CPU)."""
import numpy as np
import pytest
import torch

import oracle as O
from tests import ref_f64 as R

CASES = [
    ("top1_plain", dict(), 64, 16, 32, 4),
    ("top2_rts", dict(top_k=2, assignment_mode=O.RTS, capacity_factor_train=1.25), 96, 16, 24, 6),
    ("top1_grouped", dict(assignment_mode=O.GROUPED, group_count=2, capacity_factor_train=0.75), 64, 8, 16, 4),
    ("top2_plain_tight", dict(top_k=2, capacity_factor_train=0.5), 64, 8, 16, 4),
]


@pytest.mark.parametrize("name,kw,T,d,f,E", CASES)
def test_ref_f64_matches_restatement(name, kw, T, d, f, E):
    seed = 5
    o = O.restatement()
    x, gw, w1, b1, w2, b2, dy = O.layer_inputs(T, d, f, E, seed=seed)
    cfg = O.make_cfg(num_experts=E, **kw)
    ref = o.moe_layer(x, gw, w1, b1, w2, b2, cfg, O.TRAIN, seed, dy=dy, daux=1.0)
    probs, ch, gp, noise = o.gate_forward(x, gw, cfg, O.TRAIN, o.derive_seed(seed, "jitter"))
    assert np.array_equal(ch, ref.expert_id)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731
    out = dict(y=t(ref.y), aux=ref.aux, dx=t(ref.dx), dgate_w=t(ref.dgate_w), dw1=t(ref.dw1),
               db1=t(ref.db1), dw2=t(ref.dw2), db2=t(ref.db2))
    res = R.check_layer("cpu", out, x, gw, t(w1), t(b1), t(w2), t(b2), dy, probs=probs,
                        noise=noise, expert_id=ch, slot=ref.slot, gate_prob=gp, E=E,
                        K=kw.get("top_k", 1), alpha=0.01, daux=1.0, bf16=False)
    for k, v in res.items():
        if k.startswith("_"):
            continue
        err = v if k == "aux" else v.err
        assert err < 1e-11, (k, err)


def _emulate_bf16_device(x, gw, w1, b1, w2, b2, dy, probs, noise, ch, slot, gp, E, K, alpha):
    """The bf16 path's roundings on the CPU: H, O, dO, dH, dX stored in bf16,
    y / dx / dW returned in bf16, everything else f64 (stands in for fp32)."""
    bf = lambda a: a.to(torch.bfloat16).double()  # noqa: E731
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).double()  # noqa: E731
    X, DY, P, NZ, GW = t(x), t(dy), t(probs), t(noise), t(gw)
    T, d = X.shape
    eid = torch.from_numpy(ch.astype(np.int64)).view(T, K)
    kept = torch.from_numpy(slot.astype(np.int64)).view(T, K) >= 0
    g = torch.from_numpy(gp).view(T, K)
    w = g * E if K == 1 else g / g.sum(1, keepdim=True)
    Y = torch.zeros(T, d, dtype=torch.float64)
    dX = torch.zeros_like(Y)
    dw = torch.zeros(T, K, dtype=torch.float64)
    out = dict(dw1=torch.zeros_like(w1), dw2=torch.zeros_like(w2), db1=torch.zeros_like(b1),
               db2=torch.zeros_like(b2))
    for e in range(E):
        tt, kk = torch.nonzero((eid == e) & kept, as_tuple=True)
        Xe = X[tt]
        H = bf((Xe @ w1[e] + b1[e]).clamp_min(0))
        O_ = bf(H @ w2[e] + b2[e])
        we = w[tt, kk].unsqueeze(1)
        Y.index_put_((tt,), we * O_, accumulate=True)
        dw[tt, kk] = (DY[tt] * O_).sum(1)
        dO = bf(we * DY[tt])
        dH = bf((dO @ w2[e].T) * (H > 0))
        dX.index_put_((tt,), bf(dH @ w1[e].T), accumulate=True)
        out["dw1"][e] = bf(Xe.T @ dH)
        out["dw2"][e] = bf(H.T @ dO)
        out["db1"][e] = dH.sum(0)
        out["db2"][e] = dO.sum(0)
    none = ~kept.any(1)
    Y[none] = X[none]
    dP = torch.zeros(T, E, dtype=torch.float64)
    if K == 1:
        dP.scatter_add_(1, eid[:, :1], E * dw * kept)
    else:
        S = g.sum(1, keepdim=True)
        dk = dw * kept
        dP.scatter_add_(1, eid, dk / S - (dk * g).sum(1, keepdim=True) / (S * S))
    cnt0 = torch.bincount(eid[:, 0], minlength=E).double()
    fc = alpha * E * cnt0 / T
    dP = dP + fc / T
    dL = P * (dP - (dP * P).sum(1, keepdim=True))
    DXg = (dL @ GW.T) * NZ
    DX = dX + DXg
    DX[none] += DY[none]
    out.update(y=bf(Y), dx=bf(DX), dgate_w=(X * NZ).T @ dL, aux=float((P.mean(0) * fc).sum()))
    return out


@pytest.mark.parametrize("name,kw,T,d,f,E", CASES[:2])
def test_bf16_bound_holds_for_emulated_roundings(name, kw, T, d, f, E):
    """The derived bound is satisfied by a CPU emulation of exactly the bf16
    path's roundings, and not vacuous: the worst element sits within 1/1000 of
    the bound or closer (the emulated error is a visible fraction of it)."""
    seed = 6
    o = O.restatement()
    x, gw, w1, b1, w2, b2, dy = O.layer_inputs(T, 64, 128, E, seed=seed)
    x = torch.from_numpy(x).to(torch.bfloat16).double().numpy()
    dy = torch.from_numpy(dy).to(torch.bfloat16).double().numpy()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).double()  # noqa
    W1, W2, B1, B2 = t(w1), t(w2), torch.from_numpy(b1), torch.from_numpy(b2)
    cfg = O.make_cfg(num_experts=E, **kw)
    K = kw.get("top_k", 1)
    probs, ch, gp, noise = o.gate_forward(x, gw, cfg, O.TRAIN, o.derive_seed(seed, "jitter"))
    slot, _ = o.assign(ch, E, o.capacity(T, cfg, O.TRAIN), K, kw.get("assignment_mode", 0), 1,
                       o.derive_seed(seed, "assign"))
    out = _emulate_bf16_device(x, gw, W1, B1, W2, B2, dy, probs, noise, ch, slot, gp, E, K, 0.01)
    res = R.check_layer("cpu", out, x, gw, W1, B1, W2, B2, dy, probs=probs, noise=noise,
                        expert_id=ch, slot=slot, gate_prob=gp, E=E, K=K, alpha=0.01, daux=1.0)
    print(name, {k: v for k, v in res.items() if not k.startswith("_")})
    R.assert_within(res, name)
    for k in ("y", "dx", "dw1", "dw2"):
        assert res[k].ratio > 1e-3, (k, res[k])
