"""The float64 path (dtype MOE_F64, f64_layer.cu) against the reference's own
outputs: every golden layer config of tests/golden (computed by the reference
itself), decisions bit-exact WITHOUT margin guards needing to matter, y and
every gradient within 1e-12 of the reference (element-wise, the
gradcheck.hpp:21-24 normalisation), most outputs bit-identical."""
import numpy as np
import pytest
import torch

from tests.golden import load as G
from tests.test_gpu_parity import cfg_of, to_dev

pytestmark = pytest.mark.gpu

TOL_F64 = 1e-12


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b)))) if a.size else 0.0


def run_f64(cfg, phase, seed, inp, daux, accumulate_into=None):
    import paper_2109_10465_b200 as M
    f8 = torch.float64
    x = to_dev(inp["x"], f8)
    T, d = x.shape
    f = inp["w1"].shape[-1]
    p = M.MoeLayerParams(to_dev(inp["gate_w"], f8), to_dev(inp["w1"], f8), to_dev(inp["b1"], f8),
                         to_dev(inp["w2"], f8), to_dev(inp["b2"], f8))
    layer = M.MoeLayer(cfg_of(cfg), T, d, f, f8)
    res = None if inp.get("residual") is None else to_dev(inp["residual"], f8)
    y, aux, dec = layer.forward(x, p, M.Phase(phase), seed, residual=res)
    g = layer.backward(to_dev(inp["dy"], f8), daux, grads=accumulate_into,
                       accumulate=accumulate_into is not None)
    torch.cuda.synchronize()
    out = dict(y=y, aux=aux[0], expert_id=dec.expert_id, slot=dec.slot, gate_prob=dec.gate_prob, **g)
    return {k: (v.cpu().numpy() if torch.is_tensor(v) else v) for k, v in out.items()}


@pytest.mark.parametrize("name", G.layer_names())
def test_f64_layer_vs_reference_golden(name):
    cfg, phase, seed, daux, inp, z = G.load_layer(name)
    out = run_f64(cfg, phase, seed, inp, daux)
    assert np.array_equal(out["expert_id"].astype(np.int32), z["expert_id"])
    assert np.array_equal(out["slot"].astype(np.int32), z["slot"])
    errs = {k: rel(out[k], z[k]) for k in ("y", "gate_prob", "dx", "dgate_w", "db1", "db2", "dw1", "dw2",
                                           "dresidual") if k in z}
    errs["aux"] = rel(out["aux"], z["aux"])
    exact = float(np.mean(out["y"] == z["y"]))
    print(name, {k: f"{v:.1e}" for k, v in errs.items()}, f"y bit-identical {exact:.3f}")
    assert all(v <= TOL_F64 for v in errs.values()), errs


def test_f64_c1_full_size():
    """Config 1 at full size (T=4096, d=512, f=2048, E=8, train, jitter on)
    through the f64 path vs the reference's own outputs (c1_full.npz): no
    ReLU-kink exclusions are needed at the reference's precision."""
    import oracle as O
    from oracle.margin import margin_guard
    z = G.load_c1()
    T, d, f, E = (int(v) for v in z["spec"][:4])
    x, gw, w1, b1, w2, b2, dy = O.layer_inputs(T, d, f, E, seed=42)
    cfg = O.make_cfg(num_experts=E)
    x = margin_guard(x, gw, cfg, O.TRAIN, 42)
    out = run_f64(cfg, O.TRAIN, 42, dict(x=x, gate_w=gw, w1=w1, b1=b1, w2=w2, b2=b2, dy=dy), 1.0)
    assert np.array_equal(out["expert_id"].astype(np.int8), z["expert_id"])
    assert np.array_equal(out["slot"].astype(np.int16), z["slot"])
    rows = z["sample_rows"]
    errs = dict(y=rel(out["y"][rows], z["y_rows"]), dx=rel(out["dx"][rows], z["dx_rows"]),
                aux=rel(out["aux"], z["aux"]), dgate_w=rel(out["dgate_w"], z["dgate_w"]),
                db1=rel(out["db1"], z["db1"]), db2=rel(out["db2"], z["db2"]),
                y_rowsum=rel(out["y"].sum(1), z["y_rowsum"]),
                dw1_colsum=rel(out["dw1"].sum(1), z["dw1_colsum"]),
                dw2_rowsum=rel(out["dw2"].sum(2), z["dw2_rowsum"]))
    print({k: f"{v:.1e}" for k, v in errs.items()})
    assert all(v <= 1e-11 for v in errs.values()), errs


def test_f64_accumulate_adds_into_grads():
    """accumulate=True adds (the tape's +=, tensor.cpp:31-36): two backward
    passes into the same buffers give twice one pass."""
    name = G.layer_names()[0]
    cfg, phase, seed, daux, inp, z = G.load_layer(name)
    one = run_f64(cfg, phase, seed, inp, daux)
    acc = {k: torch.from_numpy(v).cuda().clone() for k, v in one.items()
           if k in ("dx", "dgate_w", "dw1", "db1", "dw2", "db2")}
    acc["dresidual"] = None
    two = run_f64(cfg, phase, seed, inp, daux, accumulate_into=acc)
    for k in ("dx", "dgate_w", "dw1", "db1", "dw2", "db2"):
        assert np.array_equal(two[k], 2.0 * one[k]), k
