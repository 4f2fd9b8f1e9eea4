"""Small MoE-layer fwd+bwd runs for compute-sanitizer (memcheck / racecheck /
synccheck).  Shapes are chosen so every kernel family launches: the fp32 FMA
path (gate.cu / gate2.cu / gemm_simt.cu), the bf16 tcgen05 path (gemm_tc.cu
1-CTA and CTA-pair variants, gate_tc.cu), the router / assignment / permute
kernels in plain, RTS and grouped modes, and the jitter generator.

    compute-sanitizer --tool racecheck python scripts/sanitize_layer.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_10465_b200 as M  # noqa: E402


def layer(dtype, T, d, f, E, **kw):
    g = torch.Generator(device="cpu").manual_seed(3)
    cfg = M.RouterConfig(num_experts=E, **kw)
    L = M.MoeLayer(cfg, T, d, f, dtype)
    r = lambda *s, sc=1.0: (torch.rand(*s, generator=g) * 2 - 1) * sc  # noqa: E731
    p = M.MoeLayerParams(r(d, E, sc=0.05).cuda(), r(E, d, f, sc=0.02).to("cuda", dtype),
                         r(E, f, sc=0.01).cuda(), r(E, f, d, sc=0.02).to("cuda", dtype),
                         r(E, d, sc=0.01).cuda())
    x = r(T, d).to("cuda", dtype)
    y, aux, dec = L.forward(x, p, M.Phase.TRAIN, 42)
    g_ = L.backward(r(T, d).to("cuda", dtype), 1.0)
    torch.cuda.synchronize()
    print(f"{dtype} T={T} d={d} f={f} E={E} {kw}: y {float(y.float().abs().mean()):.4f} "
          f"dx {float(g_['dx'].float().abs().mean()):.4f}", flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("all", "fp32"):
        layer(torch.float32, 512, 128, 256, 8, top_k=2, assignment_mode=M.AssignmentMode.RTS,
              capacity_factor_train=1.25)
    if which in ("all", "bf16"):
        layer(torch.bfloat16, 1024, 256, 512, 8)
        layer(torch.bfloat16, 1024, 256, 512, 4, assignment_mode=M.AssignmentMode.GROUPED,
              group_count=4, capacity_factor_train=1.5)
    if which in ("all", "pair"):  # >= 256 rows per expert -> cta_group::2 GEMMs
        layer(torch.bfloat16, 2048, 256, 512, 4)
