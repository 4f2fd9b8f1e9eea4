import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import oracle as O
from oracle.margin import margin_guard
from tests.golden import load as G
from tests.test_gpu_parity import run_gpu_layer, rel_err, rel_norm
z = G.load_c1()
T, d, f, E = (int(v) for v in z["spec"][:4])
x, gw, w1, b1, w2, b2, dy = O.layer_inputs(T, d, f, E, seed=42)
cfg = O.make_cfg(num_experts=E)
x = margin_guard(x, gw, cfg, O.TRAIN, 42)
out = run_gpu_layer(cfg, O.TRAIN, 42, dict(x=x, gate_w=gw, w1=w1, b1=b1, w2=w2, b2=b2, dy=dy), 1.0)
print("kept", out["stats"][2].tolist())
for k in ("db1", "db2"):
    a, b = out[k], z[k]
    print(k, "max|ref|", np.abs(b).max(), "per-expert maxabs err", np.abs(a - b).max(1))
    e = np.abs(a - b).max(1).argmax()
    j = np.abs(a[e] - b[e]).argmax()
    print("  worst", e, j, a[e, j], b[e, j])
print("dw1 colsum", rel_err(out["dw1"].sum(1), z["dw1_colsum"]), "dw2 rowsum", rel_err(out["dw2"].sum(2), z["dw2_rowsum"]))
print("dw1 rowsum", rel_norm(out["dw1"].sum(2), z["dw1_rowsum"]), "dw2 colsum", rel_norm(out["dw2"].sum(1), z["dw2_colsum"]))
