"""GPU parity of the bf16 tensor-core path (tcgen05 grouped GEMMs).

Decisions are bit-exact against the f64 oracle run on the same bf16-rounded
inputs (margin-guarded).  Outputs and gradients are checked element by
element against the bound derived from the path's bf16 roundings (stored H /
dH, stored O / dX, returned y / dx / dW; unit roundoff 2^-8) in
tests/ref_f64.py, at small shapes against the oracle's full layer and at the
full config-2 / config-3 sizes against an f64 recomputation from the oracle's
decisions.  The older norm-wise 2e-2 check is kept for the small cases.
"""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle as O
from oracle.margin import margin_guard

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2


def bf16_round(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).float().numpy().astype(np.float64)


def normwise(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


def set_tc(on: bool):
    from paper_2109_10465_b200 import _lib
    _lib.load().moe_debug_set_tensor_cores(1 if on else 0)


def run(cfg_kwargs, T, d, f, E, seed, arrays, phase=0, daux=1.0):
    import paper_2109_10465_b200 as M
    dev = lambda a, dt=torch.float32: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)  # noqa
    x, gw, w1, b1, w2, b2, dy = arrays
    cfg = M.RouterConfig(num_experts=E, **cfg_kwargs)
    layer = M.MoeLayer(cfg, T, d, f, torch.bfloat16)
    p = M.MoeLayerParams(dev(gw), dev(w1, torch.bfloat16), dev(b1), dev(w2, torch.bfloat16), dev(b2))
    y, aux, dec = layer.forward(dev(x, torch.bfloat16), p, M.Phase(phase), seed)
    g = layer.backward(dev(dy, torch.bfloat16), daux)
    torch.cuda.synchronize()
    out = dict(y=y, aux=aux[0], expert_id=dec.expert_id, slot=dec.slot, **g)
    return {k: (v.float().cpu().numpy() if torch.is_tensor(v) else v) for k, v in out.items()}


CASES = [
    ("top1_plain", dict(), 1024, 256, 512, 8),
    ("top2_rts_c125", dict(top_k=2, assignment_mode=2, capacity_factor_train=1.25), 1024, 256, 512, 8),
    ("top1_grouped", dict(assignment_mode=1, group_count=4, capacity_factor_train=1.5), 1024, 256, 512, 4),
    ("top1_e64", dict(), 4096, 256, 512, 64),
]


def make_inputs(T, d, f, E, seed, cfgk):
    x, gw, w1, b1, w2, b2, dy = O.layer_inputs(T, d, f, E, seed=seed)
    ocfg = O.make_cfg(num_experts=E, top_k=cfgk.get("top_k", 1),
                      assignment_mode=cfgk.get("assignment_mode", 0),
                      group_count=cfgk.get("group_count", 1),
                      capacity_factor_train=cfgk.get("capacity_factor_train", 1.0))
    x = bf16_round(x)
    x = margin_guard(x, gw, ocfg, O.TRAIN, seed, round_fn=bf16_round)
    return ocfg, [bf16_round(x), gw.astype(np.float32).astype(np.float64), bf16_round(w1),
                  b1.astype(np.float32).astype(np.float64), bf16_round(w2),
                  b2.astype(np.float32).astype(np.float64), bf16_round(dy)]


@pytest.mark.parametrize("name,cfgk,T,d,f,E", CASES)
def test_bf16_tcgen05_vs_oracle(name, cfgk, T, d, f, E):
    seed = 7
    ocfg, arrs = make_inputs(T, d, f, E, seed, cfgk)
    set_tc(True)
    out = run(cfgk, T, d, f, E, seed, arrs)
    ref = O.restatement().moe_layer(*arrs[:6], ocfg, O.TRAIN, seed, dy=arrs[6], daux=1.0)
    assert np.array_equal(out["expert_id"].astype(np.int32), ref.expert_id)
    assert np.array_equal(out["slot"].astype(np.int32), ref.slot)
    errs = {k: normwise(out[k], getattr(ref, k)) for k in ("y", "dx", "dgate_w", "dw1", "db1", "dw2", "db2")}
    errs["aux"] = abs(float(out["aux"]) - ref.aux)
    print(name, {k: f"{v:.2e}" for k, v in errs.items()})
    assert all(v <= BF16_TOL for v in errs.values()), errs
    # every element within the derived bf16 bound (tests/ref_f64.py)
    from tests import ref_f64 as R
    K = cfgk.get("top_k", 1)
    o = O.restatement()
    probs, ch, gp, noise = o.gate_forward(arrs[0], arrs[1], ocfg, O.TRAIN, o.derive_seed(seed, "jitter"))
    assert np.array_equal(ch, ref.expert_id)
    tt = lambda a, dt=torch.float32: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)  # noqa
    dout = {k: tt(v) for k, v in out.items() if k not in ("expert_id", "slot") and v is not None}
    res = R.check_layer("cuda", dout, arrs[0], arrs[1], tt(arrs[2]), tt(arrs[3]), tt(arrs[4]),
                        tt(arrs[5]), arrs[6], probs=probs, noise=noise, expert_id=ch,
                        slot=ref.slot, gate_prob=gp, E=E, K=K, alpha=0.01, daux=1.0)
    print(name, {k: v for k, v in res.items() if not k.startswith("_")})
    R.assert_within(res, name)


@pytest.mark.parametrize("name,cfgk,T,d,f,E", CASES[:2])
def test_bf16_tcgen05_vs_simt(name, cfgk, T, d, f, E):
    """Same inputs through the tcgen05 kernels and the SIMT kernels: identical
    decisions, outputs within bf16 output rounding of each other."""
    seed = 9
    _, arrs = make_inputs(T, d, f, E, seed, cfgk)
    set_tc(True)
    a = run(cfgk, T, d, f, E, seed, arrs)
    set_tc(False)
    b = run(cfgk, T, d, f, E, seed, arrs)
    set_tc(True)
    assert np.array_equal(a["slot"], b["slot"])
    errs = {k: normwise(a[k], b[k]) for k in ("y", "dx", "dw1", "dw2", "db1", "db2")}
    print(name, {k: f"{v:.2e}" for k, v in errs.items()})
    assert all(v <= 1e-2 for v in errs.values()), errs


def oracle_decisions(x, gw, ocfg, seed, T, E, K, mode, G=1):
    """Gate + assignment of the f64 restatement (routing.cpp:51-206)."""
    o = O.restatement()
    probs, ch, gp, noise = o.gate_forward(x, gw, ocfg, O.TRAIN, o.derive_seed(seed, "jitter"))
    cap = o.capacity(T, ocfg, O.TRAIN)
    slot, dcap = o.assign(ch, E, cap, K, mode, G, o.derive_seed(seed, "assign"))
    return probs, ch, gp, noise, slot, dcap


def device_layer(T, d, f, E, gen_seed, x, gw, cfg_kwargs, dev="cuda"):
    """bf16 weights drawn on the device (U(-s,s), s = sqrt(6/(d+f)); biases
    U(-.01,.01)), x/gw given (numpy f64 of bf16 / fp32 values)."""
    import paper_2109_10465_b200 as M
    g = torch.Generator(device=dev).manual_seed(gen_seed)
    s1 = float(np.sqrt(6.0 / (d + f)))
    w1 = ((torch.rand(E, d, f, device=dev, generator=g) * 2 - 1) * s1).to(torch.bfloat16)
    w2 = ((torch.rand(E, f, d, device=dev, generator=g) * 2 - 1) * s1).to(torch.bfloat16)
    b1 = (torch.rand(E, f, device=dev, generator=g) * 2 - 1) * 0.01
    b2 = (torch.rand(E, d, device=dev, generator=g) * 2 - 1) * 0.01
    dy = (torch.rand(T, d, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    p = M.MoeLayerParams(torch.from_numpy(gw.astype(np.float32)).to(dev), w1, b1, w2, b2)
    xd = torch.from_numpy(x.astype(np.float32)).to(dev).to(torch.bfloat16)
    layer = M.MoeLayer(M.RouterConfig(num_experts=E, **cfg_kwargs), T, d, f, torch.bfloat16)
    return layer, p, xd, dy


def run_full_size(T, d, f, E, seed, cfg_kwargs, mode, expect_cap, expect_drops=None):
    from tests import ref_f64 as R

    import paper_2109_10465_b200 as M
    K = cfg_kwargs.get("top_k", 1)
    x0, gw, *_ = O.layer_inputs(T, d, 8, E, seed=seed)
    gw = gw.astype(np.float32).astype(np.float64)
    ocfg = O.make_cfg(num_experts=E, top_k=K, assignment_mode=mode,
                      capacity_factor_train=cfg_kwargs.get("capacity_factor_train", 1.0))
    x = margin_guard(bf16_round(x0), gw, ocfg, O.TRAIN, seed, round_fn=bf16_round)
    layer, p, xd, dy = device_layer(T, d, f, E, seed, x, gw, cfg_kwargs)
    set_tc(True)
    assert layer.handle.gemm_path() == "tcgen05"
    y, aux, dec = layer.forward(xd, p, M.Phase.TRAIN, seed)
    g = layer.backward(dy, 1.0)
    y2, _, _ = layer.forward(xd, p, M.Phase.TRAIN, seed)   # bitwise determinism
    torch.cuda.synchronize()
    assert torch.equal(y, y2)
    probs, ch, gp, noise, slot, cap = oracle_decisions(x, gw, ocfg, seed, T, E, K, mode)
    assert cap == dec.capacity == expect_cap
    assert np.array_equal(dec.expert_id.cpu().numpy(), ch), "expert ids differ from the oracle"
    assert np.array_equal(dec.slot.cpu().numpy(), slot), "capacity slots differ from the oracle"
    if expect_drops is not None:
        assert int((slot < 0).sum()) == expect_drops
    kept = np.bincount(ch[slot >= 0], minlength=E)
    assert kept.max() <= cap
    out = dict(y=y, aux=aux[0], **g)
    res = R.check_layer("cuda", out, x, gw, p.w1, p.b1, p.w2, p.b2,
                        dy.float().cpu().numpy().astype(np.float64), probs=probs, noise=noise,
                        expert_id=ch, slot=slot, gate_prob=gp, E=E, K=K, alpha=0.01, daux=1.0)
    print({k: v for k, v in res.items() if not k.startswith("_")})
    R.assert_within(res, f"T={T} d={d} f={f} E={E} k={K}")
    return res


def test_bf16_c3_full_size():
    """Config 3 on one GPU (T=8192, d=2048, f=8192, E=64, top-1, C=1.0, plain,
    train with jitter), the bench workload: decisions bit-exact vs the f64
    oracle's gate + assignment; y, dx, dgate_w and dW1 / db1 / dW2 / db2 of
    ALL 64 experts in every element within the derived bf16 bound of an f64
    recomputation from the oracle's decisions (tests/ref_f64.py); aux within
    1e-5; two forwards bitwise identical."""
    run_full_size(8192, 2048, 8192, 64, 42, dict(), O.PLAIN, expect_cap=128)


def test_bf16_c2_full_size():
    """Config 2 at full size (T=16384, d=1024, f=4096, E=32, top-2, C=1.25,
    RTS, alpha 0.01, eps 0.01): cap 640 and exactly 12,288 of 32,768 routes
    dropped (capacity ignores top_k, routing.cpp:43-49), decisions bit-exact,
    every output and gradient element within the derived bf16 bound."""
    run_full_size(16384, 1024, 4096, 32, 11,
                  dict(top_k=2, assignment_mode=2, capacity_factor_train=1.25), O.RTS,
                  expect_cap=640, expect_drops=12288)


@pytest.mark.parametrize("pair", ["0", "1"])
def test_bf16_gemm_variants_subprocess(pair):
    """Both tcgen05 kernel variants (1-CTA and cta_group::2 CTA pairs, chosen by
    MOE_B200_PAIR) pass the bf16-vs-oracle cases, including experts with an odd
    number of 128-row tiles (the pair's second CTA then has no rows)."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, MOE_B200_PAIR=pair)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-k", "vs_oracle",
                        os.path.abspath(__file__)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("top_k,T,E", [(1, 8192, 64), (2, 1000, 64), (1, 300, 64), (1, 4096, 8),
                                       (2, 1000, 16), (1, 2048, 32), (2, 300, 32),
                                       (1, 16384, 64), (2, 12000, 16)])
def test_fused_gate_matches_split_kernels(top_k, T, E):
    _fused_gate_vs_split(top_k, T, E, "TRAIN")


@pytest.mark.parametrize("top_k,T,E", [(1, 16384, 16), (2, 1000, 16), (1, 4096, 8), (1, 40000, 16),
                                       (1, 8192, 64), (2, 3000, 32)])
def test_fused_gate_eval_matches_split_kernels(top_k, T, E):
    """Eval (no jitter): E <= 16 runs the two-CTAs-per-SM instance
    (GCfg<16, true>), as a CTA pair for T <= 148 tiles and one CTA per tile
    above; E = 32 / 64 the jitter-free ring of the one-CTA instance."""
    _fused_gate_vs_split(top_k, T, E, "EVAL")


def _fused_gate_vs_split(top_k, T, E, phase):
    """The fused gate (gate_fused.cu: logits + softmax + top-k + balance loss in
    one cluster kernel) against the split kernels (MOE_B200_GATE_FUSED=0:
    split-K logits, softmax_topk, balance_finalize) on the same inputs:
    identical decisions, probabilities / gate_prob / aux within fp32 rounding,
    including a ragged last tile (T % 128 != 0), for every expert count the
    fused kernel takes (E = 8 runs on the 16-column instance with padding)."""
    import os

    import paper_2109_10465_b200 as M
    d, f, seed = 2048, 256, 5
    x0, gw, *_ = O.layer_inputs(T, d, 8, E, seed=seed)
    ocfg = O.make_cfg(num_experts=E, top_k=top_k)
    x = margin_guard(bf16_round(x0), gw, ocfg, getattr(O, phase), seed, round_fn=bf16_round)
    outs = []
    for fused in ("1", "0"):
        os.environ["MOE_B200_GATE_FUSED"] = fused
        try:
            layer, p, xd, dy = device_layer(T, d, f, E, seed, x, gw.astype(np.float32).astype(np.float64),
                                            dict(top_k=top_k))
        finally:
            os.environ.pop("MOE_B200_GATE_FUSED", None)
        y, aux, dec = layer.forward(xd, p, getattr(M.Phase, phase), seed)
        torch.cuda.synchronize()
        outs.append((dec.expert_id.cpu(), dec.slot.cpu(), dec.gate_prob.cpu(), float(aux[0]), y.float().cpu()))
    (e1, s1, g1, a1, y1), (e0, s0, g0, a0, y0) = outs
    assert torch.equal(e1, e0) and torch.equal(s1, s0)
    # the two paths sum the d products in different orders (3xTF32 with the
    # hi.lo products in their own TMEM columns vs split-K FMA partials): a few
    # fp32 ulps of the logits, scaled by p ~ 1/E.  Both paths are held to the
    # oracle's bound by the vs_oracle / full-size tests.
    assert float((g1 - g0).abs().max()) <= (5e-6 if E == 64 else 1e-5)
    assert abs(a1 - a0) <= 1e-6 * max(1.0, abs(a0))
    assert float((y1 - y0).abs().max()) <= 2e-2 * max(1.0, float(y0.abs().max()))


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_backward_accumulate_and_fp32_weight_grads(dtype):
    """moe_backward_ex: MOE_GRAD_WEIGHTS_F32 writes the very fp32 accumulators
    the bf16 output rounds (bf16(dW_f32) == dW_bf16 bit for bit), and
    MOE_GRAD_ACCUMULATE adds every gradient into its buffer (the tape's +=,
    tensor.cpp:31-36): a second accumulating pass doubles it (exactly where
    the sum is exact, within one bf16 rounding for bf16 dW)."""
    import paper_2109_10465_b200 as M
    T, d, f, E, seed = 1024, 256, 512, 8, 3
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    g = torch.Generator(device="cuda").manual_seed(seed)
    r = lambda *s: torch.rand(*s, device="cuda", generator=g) * 2 - 1  # noqa: E731
    p = M.MoeLayerParams(r(d, E) * 0.1, (r(E, d, f) * 0.05).to(dt), r(E, f) * 0.01, (r(E, f, d) * 0.05).to(dt),
                         r(E, d) * 0.01)
    x, dy = r(T, d).to(dt), r(T, d).to(dt)
    layer = M.MoeLayer(M.RouterConfig(num_experts=E), T, d, f, dt)
    layer.forward(x, p, M.Phase.TRAIN, seed)
    g1 = {k: (v.clone() if v is not None else None) for k, v in layer.backward(dy, 1.0).items()}
    if dtype == "bf16":
        gf = layer.backward(dy, 1.0, weights_f32=True)
        assert gf["dw1"].dtype == torch.float32
        assert torch.equal(gf["dw1"].to(torch.bfloat16), g1["dw1"])
        assert torch.equal(gf["dw2"].to(torch.bfloat16), g1["dw2"])
        acc32 = {k: (v.clone() if v is not None else None) for k, v in gf.items()}
        layer.backward(dy, 1.0, grads=acc32, accumulate=True, weights_f32=True)
        assert torch.equal(acc32["dw1"], 2 * gf["dw1"]) and torch.equal(acc32["dw2"], 2 * gf["dw2"])
    acc = {k: (v.clone() if v is not None else None) for k, v in g1.items()}
    layer.backward(dy, 1.0, grads=acc, accumulate=True)
    torch.cuda.synchronize()
    for k in ("dx", "dgate_w", "db1", "db2"):
        assert torch.equal(acc[k], 2 * g1[k]), k
    for k in ("dw1", "dw2"):
        if dtype == "fp32":
            assert torch.equal(acc[k], 2 * g1[k]), k
        else:  # bf16(f + bf16(f)): within one bf16 rounding of 2 bf16(f)
            err = (acc[k].float() - 2 * g1[k].float()).abs()
            assert bool((err <= 2.0 ** -7 * acc[k].float().abs() + 1e-30).all()), k


@pytest.mark.parametrize("top_k,T,jitter,res", [(1, 8192, True, False), (2, 1000, True, True),
                                                 (1, 300, False, False), (2, 4096, False, True)])
def test_gate_backward_tma_kernels_match_previous(top_k, T, jitter, res):
    """The TMA-fed gate backward kernels (gate_bwd.cu: dWg by 3xBF16 MN-major
    tcgen05, dx persistent with tf32-rounded dL / Wg) against the kernels they
    replace (gate_tc.cu, MOE_B200_GATE_DW_TMA=0 / MOE_B200_GATE_DX_TMA=0) on
    the same forward: top-1 / top-2, with and without jitter, an explicit
    residual (dres) and ragged token counts (T % 128 != 0).  dx takes the same
    tf32 products and must agree to bf16 rounding; dWg is now more precise
    (2^-16 vs 2^-11 per operand), so it agrees to the TF32 kernel's error."""
    import os

    import paper_2109_10465_b200 as M
    d, f, E, seed = 2048, 256, 64, 9
    g = torch.Generator(device="cuda").manual_seed(seed)
    r = lambda *s: torch.rand(*s, device="cuda", generator=g) * 2 - 1  # noqa: E731
    p = M.MoeLayerParams(r(d, E) * 0.05, (r(E, d, f) * 0.05).bfloat16(), r(E, f) * 0.01,
                         (r(E, f, d) * 0.05).bfloat16(), r(E, d) * 0.01)
    x, dy = r(T, d).bfloat16(), r(T, d).bfloat16()
    resid = r(T, d).bfloat16() if res else None
    cfg = M.RouterConfig(num_experts=E, top_k=top_k, jitter_eps=0.01 if jitter else 0.0)
    outs = []
    for v in ("1", "0"):
        os.environ["MOE_B200_GATE_DW_TMA"] = v
        os.environ["MOE_B200_GATE_DX_TMA"] = v
        try:
            layer = M.MoeLayer(cfg, T, d, f, torch.bfloat16)
        finally:
            os.environ.pop("MOE_B200_GATE_DW_TMA", None)
            os.environ.pop("MOE_B200_GATE_DX_TMA", None)
        layer.forward(x, p, M.Phase.TRAIN, seed, residual=resid)
        gr = layer.backward(dy, 1.0)
        torch.cuda.synchronize()
        outs.append({k: (v_.float().cpu() if v_ is not None else None) for k, v_ in gr.items()})
    new, old = outs
    scale = float(old["dx"].abs().max())
    assert float((new["dx"] - old["dx"]).abs().max()) <= 2.0 ** -7 * scale
    if res:
        assert torch.equal(new["dresidual"], old["dresidual"])
    sw = float(old["dgate_w"].abs().max())
    assert float((new["dgate_w"] - old["dgate_w"]).abs().max()) <= 2e-3 * sw
    for k in ("dw1", "dw2", "db1", "db2"):
        assert torch.equal(new[k], old[k]), k


@pytest.mark.parametrize("top_k,T,res", [(1, 8192, False), (2, 1000, True)])
def test_router_combine_backward_fused_is_bit_identical(top_k, T, res):
    """router_combine_bwd_kernel (one pass over dy: dO rows, dw = <dy, O>, the
    routing-weight / balance / softmax backward) against the two kernels it
    replaces (MOE_B200_RCB_FUSED=0): the same operations in the same order, so
    every gradient is bit-identical."""
    import os

    import paper_2109_10465_b200 as M
    d, f, E, seed = 1024, 512, 64, 4
    g = torch.Generator(device="cuda").manual_seed(seed)
    r = lambda *s: torch.rand(*s, device="cuda", generator=g) * 2 - 1  # noqa: E731
    p = M.MoeLayerParams(r(d, E) * 0.05, (r(E, d, f) * 0.05).bfloat16(), r(E, f) * 0.01,
                         (r(E, f, d) * 0.05).bfloat16(), r(E, d) * 0.01)
    x, dy = r(T, d).bfloat16(), r(T, d).bfloat16()
    resid = r(T, d).bfloat16() if res else None
    outs = []
    for v in ("1", "0"):
        os.environ["MOE_B200_RCB_FUSED"] = v
        try:
            layer = M.MoeLayer(M.RouterConfig(num_experts=E, top_k=top_k), T, d, f, torch.bfloat16)
        finally:
            os.environ.pop("MOE_B200_RCB_FUSED", None)
        layer.forward(x, p, M.Phase.TRAIN, seed, residual=resid)
        gr = layer.backward(dy, 1.0)
        torch.cuda.synchronize()
        outs.append({k: (v_.cpu() if v_ is not None else None) for k, v_ in gr.items()})
    for k, v_ in outs[0].items():
        if v_ is not None:
            assert torch.equal(v_, outs[1][k]), k
