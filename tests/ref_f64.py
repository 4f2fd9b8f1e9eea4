"""f64 recomputation of the MoE layer from the oracle's routing decisions, with
a per-element error bound for the bf16 tensor-core path.  TEST INFRASTRUCTURE.

Decisions (expert ids, slots, capacity) and the f64 jitter noise and
probabilities come from the C restatement (oracle/moe_oracle.c, pinned to the
reference).  Given them, the floating-point part of the layer is dense
algebra; this module evaluates it in float64 on the GPU (cuBLAS DGEMM) so the
headline shapes (config 3: T=8192, d=2048, f=8192, E=64; config 2 at full
size) can be checked in every element instead of sampled rows.  It follows
the reference's formulas line by line:

  forward   routing.cpp:397-424  H = relu(X W1 + b1), O = H W2 + b2,
                                 y = sum_k w_k O_k (w = E p top-1; p_k/(p0+p1) top-2),
                                 dropped-everywhere tokens y = residual
            routing.cpp:348-374  aux = sum_e mean_t P[t,e] * alpha E cnt0_e / T
  backward  routing.cpp:311-344 (combine), ops.cpp:135-144 (matmul), 199-209 (bias),
            307-315 (relu), 329-343 (softmax), 213-235 (jitter mul), 250-262 (div),
            528-537 / 552-558 (balance), 579-585 (pick)

Error bound of the bf16 path.  The device rounds to bf16
(8-bit significand, unit roundoff u = 2^-8, round-to-nearest-even) in three
places along each chain: the stored hidden activations H and dH, the stored
expert outputs O and input-gradients dX, and the returned tensors (y, dx,
dW1, dW2).  Every other quantity is fp32 (accumulators, logits, probabilities,
gate gradients).  For an element Z = sum_j a_j b_j whose operands carry
independent relative rounding errors |delta_j| <= u, Var(dZ) <= (u^2/3)
sum_j (a_j b_j)^2 (uniform rounding errors), which propagates through the
linear chain; a rounding of Z itself is bounded deterministically by u |Z|.
The asserted bound per element is

    |gpu - f64| <= SIG * sqrt(Var) + det + FLOOR * max|f64 tensor|

with SIG = 8 standard deviations (the summed errors are bounded, lighter
tailed than a Gaussian; 8 sigma is < 1e-15 per element even as a Gaussian)
and FLOOR = 1e-5 for fp32 accumulation and the fp32 gate (3xTF32 logits are
accurate to ~1e-6 relative).
"""
from __future__ import annotations

import numpy as np
import torch

U = 2.0 ** -8
SIG = 8.0
FLOOR = 1e-5
V = U * U / 3.0  # variance of one bf16 rounding, relative


class Stat:
    """max |dev - ref|, max ratio to the bound, norm-wise error.  Each piece
    (a whole tensor, or one expert's slice) is checked against its own bound
    with the floor scaled by that piece's max |ref|."""

    def __init__(self):
        self.err = 0.0
        self.ratio = 0.0
        self.refmax = 0.0

    def add(self, dev, ref, var, det=None):
        diff = (dev.double() - ref).abs()
        if diff.numel() == 0:
            return
        rmax = float(ref.abs().max())
        self.err = max(self.err, float(diff.max()))
        self.refmax = max(self.refmax, rmax)
        bound = SIG * var.clamp_min(0).sqrt() + FLOOR * max(1.0, rmax)
        if det is not None:
            bound = bound + det
        self.ratio = max(self.ratio, float((diff / bound).max()))

    def normwise(self):
        return self.err / max(1.0, self.refmax)

    def __repr__(self):
        return f"err {self.err:.2e} norm {self.normwise():.2e} bound-ratio {self.ratio:.3f}"


def check_layer(dev, out, x, gw, w1, b1, w2, b2, dy, *, probs, noise, expert_id, slot, gate_prob,
                E, K, alpha, daux, residual=None, bf16=True, experts=None, expert_sink=None):
    """Compare the device outputs ``out`` (dict of torch tensors: y, aux, dx,
    dgate_w, dw1, db1, dw2, db2[, dresidual]) of one layer call against the
    f64 recomputation.  x, dy, gw, noise, probs: numpy f64 (values as the GPU
    saw them); w1/w2/b1/b2: the device tensors themselves (their values are
    the inputs).  Returns {name: Stat}; ratios <= 1 mean within the bound.
    ``experts`` restricts the expert-gradient comparison (all by default).
    Expert parallelism (parallel.cpp:231-366, backward by composition): with
    ``expert_sink`` the per-expert gradient contributions of these tokens are
    handed to ``expert_sink(e, {name: (ref, var)})`` instead of compared (the
    owner sums them over origin ranks); with ``out=None`` nothing is compared
    and the result holds only "_dgate_w": (ref, var) for the sum over ranks."""
    f64 = torch.float64
    T, d = x.shape
    u_on = 1.0 if bf16 else 0.0
    X = torch.from_numpy(np.ascontiguousarray(x)).to(dev, f64)
    DY = torch.from_numpy(np.ascontiguousarray(dy)).to(dev, f64)
    GW = torch.from_numpy(np.ascontiguousarray(gw)).to(dev, f64)
    P = torch.from_numpy(np.ascontiguousarray(probs)).to(dev, f64)
    NZ = None if noise is None else torch.from_numpy(np.ascontiguousarray(noise)).to(dev, f64)
    eid = torch.from_numpy(np.asarray(expert_id, np.int64)).to(dev).view(T, K)
    sl = torch.from_numpy(np.asarray(slot, np.int64)).to(dev).view(T, K)
    gp = torch.from_numpy(np.asarray(gate_prob, np.float64)).to(dev).view(T, K)
    kept = sl >= 0
    # combine weights, routing.cpp:408-417
    if K == 1:
        w = gp * E
    else:
        S = gp.sum(1, keepdim=True)
        w = gp / S
    Y = torch.zeros(T, d, dtype=f64, device=dev)
    varY = torch.zeros_like(Y)
    detY = torch.zeros_like(Y)
    dX = torch.zeros(T, d, dtype=f64, device=dev)
    var_dX = torch.zeros_like(dX)
    det_dX = torch.zeros_like(dX)
    dw = torch.zeros(T, K, dtype=f64, device=dev)     # <dy, O> per kept route
    var_dw = torch.zeros_like(dw)
    st = {k: Stat() for k in ("y", "dx", "dgate_w", "dw1", "db1", "dw2", "db2")}
    ex = range(E) if experts is None else experts
    exset = set(ex)
    for e in range(E):
        tk = (eid == e) & kept
        if not bool(tk.any()) and e not in exset:
            continue
        tt, kk = torch.nonzero(tk, as_tuple=True)
        W1 = w1[e].to(f64)
        W2 = w2[e].to(f64)
        B1 = b1[e].to(f64)
        B2 = b2[e].to(f64)
        Xe = X[tt]
        Hpre = Xe @ W1 + B1
        H = Hpre.clamp_min(0)
        O = H @ W2 + B2
        we = w[tt, kk].unsqueeze(1)
        # O error: H stored bf16 (statistical through W2), O stored bf16 (deterministic)
        varO = u_on * V * ((H * H) @ (W2 * W2))
        detO = u_on * U * O.abs()
        Y.index_put_((tt,), we * O, accumulate=True)
        varY.index_put_((tt,), we * we * varO, accumulate=True)
        detY.index_put_((tt,), we * detO, accumulate=True)
        dw[tt, kk] = (DY[tt] * O).sum(1)
        var_dw[tt, kk] = (DY[tt] ** 2 * (varO + u_on * V * O * O)).sum(1)
        # backward, ops.cpp:135-144 / 199-209 / 307-315
        dO = we * DY[tt]                                   # stored bf16 (det u|dO|)
        mask = (Hpre > 0).to(f64)
        dHu = dO @ W2.T
        dHpre = dHu * mask
        var_dH = u_on * V * (((dO * dO) @ (W2 * W2).T) * mask + dHpre * dHpre)  # dO and dH roundings
        # ReLU kink (ops.cpp:307-315): where |Hpre| is within the device's fp32
        # accumulation error of 0, its mask may differ; allow the full dH there
        amb = Hpre.abs() <= 3e-5 * ((Xe * Xe) @ (W1 * W1) + B1 * B1).sqrt()
        var_dH = var_dH + amb * dHu * dHu
        dXe = dHpre @ W1.T
        dX.index_put_((tt,), dXe, accumulate=True)
        var_dX.index_put_((tt,), var_dH @ (W1 * W1).T, accumulate=True)
        det_dX.index_put_((tt,), u_on * U * dXe.abs(), accumulate=True)   # dX stored bf16
        if e in exset and expert_sink is not None:
            expert_sink(e, dict(dw1=(Xe.T @ dHpre, (Xe * Xe).T @ var_dH),
                                dw2=(H.T @ dO, u_on * V * ((H * H).T @ (dO * dO) * 2.0)),
                                db1=(dHpre.sum(0), var_dH.sum(0)),
                                db2=(dO.sum(0), u_on * V * (dO * dO).sum(0))))
        elif e in exset and out is not None:
            dW1 = Xe.T @ dHpre
            dW2 = H.T @ dO
            db1 = dHpre.sum(0)
            db2 = dO.sum(0)
            g = out["dw1"][e]
            st["dw1"].add(g, dW1, (Xe * Xe).T @ var_dH, u_on * U * dW1.abs())
            st["dw2"].add(out["dw2"][e], dW2,
                          u_on * V * ((H * H).T @ (dO * dO) * 2.0), u_on * U * dW2.abs())
            st["db1"].add(out["db1"][e], db1, var_dH.sum(0))
            st["db2"].add(out["db2"][e], db2, u_on * V * (dO * dO).sum(0))
        del W1, W2, Hpre, H, O
    none_kept = ~kept.any(1)
    RES = X if residual is None else torch.from_numpy(np.ascontiguousarray(residual)).to(dev, f64)
    Y[none_kept] = RES[none_kept]
    detY = detY + u_on * U * Y.abs()                       # y returned in bf16
    # balance loss, routing.cpp:348-374 (first choices, drops included)
    cnt0 = torch.bincount(eid[:, 0], minlength=E).to(f64)
    fcoef = alpha * E * cnt0 / T
    aux = float((P.mean(0) * fcoef).sum())
    # combine / weight / softmax backward -> dL (ops.cpp:250-262, 276-281, 329-343, 579-585)
    dP = torch.zeros(T, E, dtype=f64, device=dev)
    var_dP = torch.zeros_like(dP)
    dwk = dw * kept
    vwk = var_dw * kept
    if K == 1:
        dP.scatter_add_(1, eid[:, :1], E * dwk)
        var_dP.scatter_add_(1, eid[:, :1], E * E * vwk)
    else:
        S = gp.sum(1, keepdim=True)
        dS = -(dwk * gp).sum(1, keepdim=True) / (S * S)
        dp = dwk / S + dS
        dP.scatter_add_(1, eid, dp)
        vS = (vwk * (gp / (S * S)) ** 2).sum(1, keepdim=True)
        var_dP.scatter_add_(1, eid, vwk / (S * S) + vS)
    dP = dP + daux * fcoef / T
    dL = P * (dP - (dP * P).sum(1, keepdim=True))
    var_dL = P * P * (var_dP + (var_dP * P * P).sum(1, keepdim=True))
    G = X * NZ if NZ is not None else X
    dWg = G.T @ dL
    var_dWg = (G * G).T @ var_dL
    dxg = dL @ GW.T
    var_dxg = var_dL @ (GW * GW).T
    if NZ is not None:
        dxg = dxg * NZ
        var_dxg = var_dxg * NZ * NZ
    DX = dX + dxg
    if residual is None:
        DX[none_kept] += DY[none_kept]
    var_DX = var_dX + var_dxg
    det_DX = det_dX + u_on * U * DX.abs()                  # dx returned in bf16
    if out is None:
        return {"_dgate_w": (dWg, var_dWg)}
    st["y"].add(out["y"], Y, varY, detY)
    st["dx"].add(out["dx"], DX, var_DX, det_DX)
    st["dgate_w"].add(out["dgate_w"], dWg, var_dWg)
    res = {k: v for k, v in st.items() if v.refmax > 0 or v.err > 0 or k in ("y", "dx", "dgate_w")}
    res["_dgate_w"] = (dWg, var_dWg)
    res["aux"] = abs(float(out["aux"]) - aux) / max(1.0, abs(aux))
    if residual is not None and "dresidual" in out:
        dres = torch.zeros_like(DY)
        dres[none_kept] = DY[none_kept]
        s = Stat()
        s.add(out["dresidual"], dres, torch.zeros_like(dres))
        res["dresidual"] = s
    return res


def assert_within(res, what=""):
    bad = {k: v for k, v in res.items()
           if not k.startswith("_") and (v > 1e-5 if k == "aux" else v.ratio > 1.0)}
    assert not bad, f"{what}: outside the derived bf16 bound: {bad}"
