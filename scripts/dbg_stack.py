import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import test_gpu_stack as t
import oracle as O
from oracle.margin import margin_guard
import paper_2109_10465_b200 as M
from paper_2109_10465_b200.stack import MoeStack
T, d, f, E, nl, seed = 256, 64, 128, 8, 3, 1234
cfg_o = O.make_cfg(num_experts=E, capacity_factor_train=1.0)
o = O.restatement()
layers = []
for l in range(nl):
    x, gw, w1, b1, w2, b2, dy = O.layer_inputs(T, d, f, E, seed=100 + l)
    layers.append(tuple(a.astype(np.float32).astype(np.float64) for a in (gw, w1, b1, w2, b2)))
    if l == 0:
        x0 = x.astype(np.float32).astype(np.float64); dy0 = dy.astype(np.float32).astype(np.float64)
x0 = margin_guard(x0, layers[0][0], cfg_o, O.TRAIN, o.derive_seed(seed, 0))
xs, refs, aux, dx_ref, grads_ref = t._ref_stack(x0, layers, cfg_o, seed, dy0)
to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().float()
params = [M.MoeLayerParams(to(gw), to(w1), to(b1), to(w2), to(b2)) for gw, w1, b1, w2, b2 in layers]
st = MoeStack(M.RouterConfig(num_experts=E), nl, T, d, f, torch.float32)
out, aux_g, decs = st.forward(to(x0), params, M.Phase.TRAIN, seed)
dx, grads = st.backward(to(dy0), 1.0)
a = dx.cpu().numpy().astype(np.float64)
err = np.abs(a - dx_ref) / np.maximum(1, np.abs(dx_ref))
i = np.unravel_index(np.argmax(err), err.shape)
print("dx max rel", err.max(), "at", i, a[i], dx_ref[i], "normwise", np.abs(a-dx_ref).max()/np.abs(dx_ref).max(), "max|ref|", np.abs(dx_ref).max())
print("rows with err>1e-5:", np.unique(np.nonzero(err > 1e-5)[0])[:20])
for l in range(nl):
    for k in ("dw1","dw2","db1","db2","dgate_w"):
        g = grads[l][k].cpu().numpy().astype(np.float64); r = getattr(grads_ref[l], k)
        print(l, k, np.abs(g-r).max()/max(1, np.abs(r).max()))
# per-layer dx check: layer l's own dx given the same incoming gradient
