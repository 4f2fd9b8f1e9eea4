"""Generate golden vectors from the REFERENCE ITSELF (oracle/_ref, compiled from
/root/reference/proj/core/src by oracle/Makefile).  Run in the build container,
where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures pin both the C restatement (tests/test_oracle.py) and the GPU
path (tests/test_gpu_parity.py).  Inputs are stored with the outputs so the
fixtures are self-contained.  Large configs store decisions plus size-
independent checksums only.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402
from oracle.margin import margin_guard  # noqa: E402

# name: (T, d, f, E, top_k, mode, groups, C_train, phase, seed, residual_zero)
LAYER_CASES = {
    "top1_plain_train": (64, 32, 48, 8, 1, O.PLAIN, 1, 1.0, O.TRAIN, 11, False),
    "top1_plain_tight": (64, 32, 48, 8, 1, O.PLAIN, 1, 0.5, O.TRAIN, 12, False),
    "top2_rts_train": (96, 32, 40, 8, 2, O.RTS, 1, 1.25, O.TRAIN, 13, False),
    "top1_grouped4": (64, 16, 24, 4, 1, O.GROUPED, 4, 1.0, O.TRAIN, 14, False),
    "top2_grouped2": (64, 16, 24, 4, 2, O.GROUPED, 2, 1.5, O.TRAIN, 15, False),
    "top2_eval": (48, 16, 32, 4, 2, O.RTS, 1, 1.0, O.EVAL, 16, False),
    "top1_rts_zero_residual": (64, 24, 32, 8, 1, O.RTS, 1, 0.75, O.TRAIN, 17, True),
    "single_expert": (9, 6, 12, 1, 1, O.PLAIN, 1, 1.0, O.TRAIN, 18, False),
    "c2_shape_small": (256, 32, 64, 32, 2, O.RTS, 1, 1.25, O.TRAIN, 19, False),
    "top1_e64_small": (512, 32, 48, 64, 1, O.PLAIN, 1, 1.0, O.TRAIN, 20, False),
}

EP_CASES = {
    # name: (ep, T, d, f, E, mode, phase, seed)
    "ep2_e4_rts": (2, 9, 5, 8, 4, O.RTS, O.TRAIN, 7),
    "ep4_e8_plain_eval": (4, 16, 8, 12, 8, O.PLAIN, O.EVAL, 8),
    "ep8_e64_train": (8, 64, 16, 24, 64, O.PLAIN, O.TRAIN, 9),
}


def layer_case(ref, name, spec):
    T, d, f, E, K, mode, G, C, phase, seed, rzero = spec
    cfg = O.make_cfg(num_experts=E, top_k=K, assignment_mode=mode, group_count=G,
                     capacity_factor_train=C)
    x, gw, w1, b1, w2, b2, dy = O.layer_inputs(T, d, f, E, seed=seed)
    x = margin_guard(x, gw, cfg, phase, seed)
    res = np.zeros_like(x) if rzero else None
    out = ref.moe_layer(x, gw, w1, b1, w2, b2, cfg, phase, seed, residual=res, dy=dy, daux=0.5)
    # Weights are not stored: O.layer_inputs(T, d, f, E, seed) regenerates
    # them bit-exactly (w_checksum pins that); x is stored (margin-guarded).
    arrays = dict(x=x, y=out.y, w_checksum=np.array([a.sum() for a in (gw, w1, b1, w2, b2, dy)]),
                  aux=np.float64(out.aux), expert_id=out.expert_id, slot=out.slot,
                  gate_prob=out.gate_prob, capacity=np.int64(out.capacity), dx=out.dx,
                  dgate_w=out.dgate_w, db1=out.db1, db2=out.db2,
                  spec=np.array([T, d, f, E, K, mode, G, phase, seed, int(rzero)], np.int64),
                  cf=np.float64(C), daux=np.float64(0.5))
    if out.dw1.size <= 32768:
        arrays.update(dw1=out.dw1, dw2=out.dw2)
    else:  # size-independent checksums for the large expert-weight grads
        arrays.update(dw1_rowsum=out.dw1.sum(2), dw1_colsum=out.dw1.sum(1),
                      dw2_rowsum=out.dw2.sum(2), dw2_colsum=out.dw2.sum(1))
    if rzero:
        arrays["dresidual"] = out.dresidual
    np.savez_compressed(os.path.join(HERE, f"layer_{name}.npz"), **arrays)
    print(name, "cap", out.capacity, "drops", int((out.slot < 0).sum()), "aux", out.aux)


def ep_case(ref, name, spec):
    ep, T, d, f, E, mode, phase, seed = spec
    cfg = O.make_cfg(num_experts=E, assignment_mode=mode)
    x, gw, w1, b1, w2, b2, _ = O.layer_inputs(T * ep, d, f, E, seed=seed)
    xs = x.reshape(ep, T, d).copy()
    o = O.restatement()
    for r in range(ep):  # per-rank layer seed derive_seed(seed, r), parallel.cpp:272
        xs[r] = margin_guard(xs[r], gw, cfg, phase, o.derive_seed(seed, r))
    ys, eid, slot, gp, cap, traffic = ref.ep_forward(xs, gw, w1, b1, w2, b2, cfg, phase, seed)
    np.savez_compressed(os.path.join(HERE, f"ep_{name}.npz"), xs=xs, ys=ys, expert_id=eid, slot=slot, gate_prob=gp,
                        capacity=np.int64(cap), traffic=traffic,
                        spec=np.array([ep, T, d, f, E, mode, phase, seed], np.int64))
    print(name, "cap", cap, "drops", int((slot < 0).sum()))


def c1_full(ref):
    """Config 1 at full size (T=4096, d=512, f=2048, E=8, top-1, C=1.0, plain,
    train phase with jitter).  Stores decisions + per-row checksums."""
    T, d, f, E = 4096, 512, 2048, 8
    seed = 42
    cfg = O.make_cfg(num_experts=E)
    x, gw, w1, b1, w2, b2, dy = O.layer_inputs(T, d, f, E, seed=seed)
    x = margin_guard(x, gw, cfg, O.TRAIN, seed)
    out = ref.moe_layer(x, gw, w1, b1, w2, b2, cfg, O.TRAIN, seed, dy=dy, daux=1.0)
    rows = np.arange(0, T, 97)
    np.savez_compressed(
        os.path.join(HERE, "c1_full.npz"),
        spec=np.array([T, d, f, E, 1, O.PLAIN, 1, O.TRAIN, seed, 0], np.int64),
        x_rowsum=x.sum(1), expert_id=out.expert_id.astype(np.int8), slot=out.slot.astype(np.int16),
        gate_prob=out.gate_prob, capacity=np.int64(out.capacity), aux=np.float64(out.aux),
        y_rowsum=out.y.sum(1), y_rows=out.y[rows], sample_rows=rows,
        dx_rowsum=out.dx.sum(1), dx_rows=out.dx[rows], dgate_w=out.dgate_w,
        db1=out.db1, db2=out.db2, dw1_colsum=out.dw1.sum(1), dw2_colsum=out.dw2.sum(1),
        dw1_rowsum=out.dw1.sum(2), dw2_rowsum=out.dw2.sum(2))
    print("c1_full cap", out.capacity, "drops", int((out.slot < 0).sum()), "aux", out.aux)


if __name__ == "__main__":
    if not O.have_reference():
        sys.exit("build the reference first: make -C oracle ref")
    ref = O.reference()
    for n, s in LAYER_CASES.items():
        layer_case(ref, n, s)
    for n, s in EP_CASES.items():
        ep_case(ref, n, s)
    if "--no-c1" not in sys.argv:
        c1_full(ref)
