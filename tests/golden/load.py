"""Load golden fixtures written by make_golden.py (inputs regenerated from seeds)."""
from __future__ import annotations

import glob
import os

import numpy as np

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))


def layer_names():
    return sorted(os.path.basename(p)[6:-4] for p in glob.glob(os.path.join(HERE, "layer_*.npz")))


def ep_names():
    return sorted(os.path.basename(p)[3:-4] for p in glob.glob(os.path.join(HERE, "ep_*.npz")))


def load_layer(name):
    z = dict(np.load(os.path.join(HERE, f"layer_{name}.npz")))
    T, d, f, E, K, mode, G, phase, seed, rzero = (int(v) for v in z["spec"])
    _, gw, w1, b1, w2, b2, dy = O.layer_inputs(T, d, f, E, seed=seed)
    chk = np.array([a.sum() for a in (gw, w1, b1, w2, b2, dy)])
    assert np.array_equal(chk, z["w_checksum"]), "regenerated weights differ from the fixture's"
    cfg = O.make_cfg(num_experts=E, top_k=K, assignment_mode=mode, group_count=G,
                     capacity_factor_train=float(z["cf"]))
    inputs = dict(x=z["x"], gate_w=gw, w1=w1, b1=b1, w2=w2, b2=b2, dy=dy,
                  residual=np.zeros_like(z["x"]) if rzero else None)
    return cfg, phase, seed, float(z["daux"]), inputs, z


def load_ep(name):
    z = dict(np.load(os.path.join(HERE, f"ep_{name}.npz")))
    ep, T, d, f, E, mode, phase, seed = (int(v) for v in z["spec"])
    _, gw, w1, b1, w2, b2, _ = O.layer_inputs(T * ep, d, f, E, seed=seed)
    cfg = O.make_cfg(num_experts=E, assignment_mode=mode)
    return cfg, phase, seed, dict(xs=z["xs"], gate_w=gw, w1=w1, b1=b1, w2=w2, b2=b2), z


def load_c1():
    return dict(np.load(os.path.join(HERE, "c1_full.npz")))
