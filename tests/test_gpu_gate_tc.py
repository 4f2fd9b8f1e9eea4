"""Tensor-core gate GEMMs (gate_tc.cu, kind::tf32) against float64 torch on
the same inputs: logits (3xTF32, must match fp32-FMA accuracy: the logits
decide routing, routing.cpp:62-71), dWg and the fused dx assembly (single
TF32, ops.cpp:137-138, 223-228; they feed bf16 tensors / fp32 weight grads)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2109_10465_b200 import _lib as L
    return L.load()


def _p(t):
    return C.c_void_p(t.data_ptr())


@pytest.mark.parametrize("T,d,splits,jitter", [(256, 256, 1, True), (1000, 512, 4, True),
                                               (8192, 2048, 2, True), (300, 256, 2, False)])
def test_gate_tc_logits(T, d, splits, jitter):
    import torch
    g = torch.Generator(device="cuda").manual_seed(T + d)
    E = 64
    x = (torch.rand(T, d, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    noise = (1 + 0.01 * (torch.rand(T, d, device="cuda", generator=g) * 2 - 1)) if jitter else None
    wg = torch.randn(d, E, device="cuda", generator=g) * 0.05
    out = torch.empty(splits, T, E, device="cuda")
    st = _lib().moe_debug_gate_tc_logits(_p(x), _p(noise) if jitter else None, _p(wg), _p(out), T, d, E, splits)
    assert st == 0
    xn = x.double() * (noise.float().double() if jitter else 1.0)
    ref = xn @ wg.double()
    got = out.double().sum(0)
    err = (got - ref).abs().max().item()
    scale = ref.abs().max().item()
    # 3xTF32 with fp32 tensor-core accumulation: a few 1e-6 of max|L|, an order
    # of magnitude inside the decision margin guard (1e-4 max|L|, oracle/margin.py);
    # single TF32 would be ~1e-3
    assert err <= 1e-5 * scale, (err / scale, scale)


@pytest.mark.parametrize("T,d,splits", [(256, 256, 1), (1000, 512, 3), (8192, 2048, 16)])
def test_gate_tc_dw(T, d, splits):
    import torch
    g = torch.Generator(device="cuda").manual_seed(2 * T + d)
    E = 64
    x = (torch.rand(T, d, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    noise = 1 + 0.01 * (torch.rand(T, d, device="cuda", generator=g) * 2 - 1)
    dL = torch.randn(T, E, device="cuda", generator=g) * 1e-3
    part = torch.empty(splits, d, E, device="cuda")
    assert _lib().moe_debug_gate_tc_dw(_p(x), _p(noise), _p(dL), _p(part), T, d, E, splits) == 0
    ref = (x.double() * noise.double()).T @ dL.double()
    got = part.double().sum(0)
    rel = ((got - ref).norm() / ref.norm()).item()
    assert rel < 2e-3, rel


@pytest.mark.parametrize("T,d,K,residual_is_x", [(256, 256, 1, True), (1000, 512, 2, False),
                                                 (4096, 2048, 1, True)])
def test_gate_tc_dx(T, d, K, residual_is_x):
    import torch
    g = torch.Generator(device="cuda").manual_seed(3 * T + d)
    E, cap_pad = 64, 256
    dL = torch.randn(T, E, device="cuda", generator=g) * 1e-2
    wg = torch.randn(d, E, device="cuda", generator=g) * 0.05
    noise = 1 + 0.01 * (torch.rand(T, d, device="cuda", generator=g) * 2 - 1)
    dX = torch.randn(E * cap_pad, d, device="cuda", generator=g).to(torch.bfloat16)
    dy = torch.randn(T, d, device="cuda", generator=g).to(torch.bfloat16)
    choice = torch.randint(0, E, (T, K), device="cuda", generator=g, dtype=torch.int32)
    pos = torch.randint(-1, cap_pad, (T, K), device="cuda", generator=g, dtype=torch.int32)
    dx = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
    dres = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
    st = _lib().moe_debug_gate_tc_dx(T, d, E, K, cap_pad, _p(dL), _p(wg), _p(noise), _p(dX), _p(choice),
                                     _p(pos), _p(dy), int(residual_is_x), _p(dx), _p(dres))
    assert st == 0
    ref = (dL.double() @ wg.double().T) * noise.double()
    kept = pos >= 0
    for k in range(K):
        rows = (choice[:, k].long() * cap_pad + pos[:, k].long()).clamp(min=0)
        ref += torch.where(kept[:, k:k + 1], dX[rows].double(), torch.zeros((), dtype=torch.float64, device="cuda"))
    none = ~kept.any(1, keepdim=True)
    if residual_is_x:
        ref += torch.where(none, dy.double(), torch.zeros((), dtype=torch.float64, device="cuda"))
    else:
        rres = torch.where(none, dy.double(), torch.zeros((), dtype=torch.float64, device="cuda"))
        assert torch.equal(dres.double(), rres.to(torch.bfloat16).double())
    err = (dx.double() - ref).abs()
    assert (err <= 1e-2 * ref.abs() + 2e-3).all(), err.max().item()
