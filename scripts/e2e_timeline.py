"""Per-step timeline of bench.py's e2e leg (config 3, one GPU): when each
step's input copies run on the copy stream and when its compute runs, from
CUDA events, to see whether the copies are slow or the compute is slowed."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_2109_10465_b200 as M  # noqa: E402

dev = torch.device("cuda", 0)
E, d, f, T = 64, 2048, 8192, 8192
cfg = M.RouterConfig(num_experts=E, capacity_factor_train=1.0, jitter_eps=0.01, balance_coeff=0.01)
layer = M.MoeLayer(cfg, T, d, f, torch.bfloat16)
g = torch.Generator(device=dev).manual_seed(1)
r = lambda *s: torch.rand(*s, device=dev, generator=g) * 2 - 1  # noqa: E731
p = M.MoeLayerParams(r(d, E) * 0.05, (r(E, d, f) * 0.02).bfloat16(), r(E, f) * 0.01,
                     (r(E, f, d) * 0.02).bfloat16(), r(E, d) * 0.01)
x, dy = r(T, d).bfloat16(), r(T, d).bfloat16()
x_h, dy_h = x.cpu().pin_memory(), dy.cpu().pin_memory()
xb, dyb = [x.clone() for _ in range(2)], [dy.clone() for _ in range(2)]
y = torch.empty_like(x)
auxb = [torch.empty(1, device=dev) for _ in range(2)]
aux_h = [torch.empty(1).pin_memory() for _ in range(2)]
gb = [dict(dx=torch.empty_like(x), dgate_w=torch.empty(d, E, device=dev),
           dw1=torch.empty(E, d, f, device=dev, dtype=torch.bfloat16), db1=torch.empty(E, f, device=dev),
           dw2=torch.empty(E, f, d, device=dev, dtype=torch.bfloat16), db2=torch.empty(E, d, device=dev),
           dresidual=None) for _ in range(2)]
st = torch.cuda.current_stream()
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
done = [torch.cuda.Event() for _ in range(2)]
for ev in done:
    ev.record(st)
mode = sys.argv[1] if len(sys.argv) > 1 else "copy"
ev = []


def E_():
    return torch.cuda.Event(enable_timing=True)


def step(i):
    b = i % 2
    c0, c1, c2, k0, k1 = E_(), E_(), E_(), E_(), E_()
    with torch.cuda.stream(s_in):
        s_in.wait_event(done[b])
        c0.record(s_in)
        if mode == "copy":
            xb[b].copy_(x_h, non_blocking=True)
        c1.record(s_in)
        if mode == "copy":
            dyb[b].copy_(dy_h, non_blocking=True)
        c2.record(s_in)
    st.wait_event(c1)
    k0.record(st)
    layer.prefetch_jitter(M.derive_seed(7, i + 1), T)
    layer.forward(xb[b], p, M.Phase.TRAIN, M.derive_seed(7, i), y=y, aux=auxb[b], decision=False, check=False)
    st.wait_event(c2)
    layer.backward(dyb[b], 1.0, check=False, grads=gb[b])
    k1.record(st)
    with torch.cuda.stream(s_out):
        s_out.wait_event(k1)
        aux_h[b].copy_(auxb[b], non_blocking=True)
        done[b].record(s_out)
    ev.append((c0, c1, c2, k0, k1))


for i in range(25):
    step(i)
torch.cuda.synchronize()
t0 = ev[5][3]
print(f"mode={mode}: step  copy_x(start,ms) copy_dy(ms)  compute(start,ms)")
for i in range(5, 25):
    c0, c1, c2, k0, k1 = ev[i]
    print(f"{i:3d}  {t0.elapsed_time(c0):8.3f} {c0.elapsed_time(c1):6.3f} {c1.elapsed_time(c2):6.3f}   "
          f"{t0.elapsed_time(k0):8.3f} {k0.elapsed_time(k1):6.3f}")
print("mean step", (ev[5][3].elapsed_time(ev[24][4])) / 20)
