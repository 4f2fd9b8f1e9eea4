"""Margin guard for decision parity (SURVEY.md §7 hard part #1, §8d).

The reference routes on f64 softmax probabilities with strict ``>`` and
lowest-index ties (routing.cpp:75-92).  A GPU computing logits in fp32 can
flip a near-tie, and because slot assignment is an order-dependent scan a
single flip cascades.  Synthetic inputs are therefore margin-guarded: rows
whose f64 top-1/top-2 logit gap (and, for top-2, the 2nd/3rd gap) is below
``rel_delta * max|L|`` are re-drawn from a row-specific derived seed until
none remain.  The jitter noise is indexed by element position (routing.cpp:
64-68), so re-drawing a row leaves the noise stream unchanged.
TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import numpy as np

from . import TRAIN, Cfg, restatement, uniform


def jitter_noise(T: int, d: int, cfg: Cfg, phase: int, layer_seed: int) -> np.ndarray | None:
    if phase != TRAIN or cfg.jitter_eps <= 0.0:
        return None
    o = restatement()
    js = o.derive_seed(layer_seed, "jitter")
    return uniform(js, T * d, 1.0 - cfg.jitter_eps, 1.0 + cfg.jitter_eps).reshape(T, d)


def gaps(x, gate_w, cfg: Cfg, phase: int, layer_seed: int) -> np.ndarray:
    T, d = x.shape
    n = jitter_noise(T, d, cfg, phase, layer_seed)
    g = x * n if n is not None else x
    L = g @ gate_w
    if L.shape[1] == 1:
        return np.full(T, np.inf), 1.0
    s = np.sort(L, axis=1)[:, ::-1]
    gap = s[:, 0] - s[:, 1]
    if cfg.top_k == 2 and L.shape[1] > 2:
        gap = np.minimum(gap, s[:, 1] - s[:, 2])
    return gap, float(np.abs(L).max())


def margin_guard(x, gate_w, cfg: Cfg, phase: int, layer_seed: int, rel_delta: float = 1e-4,
                 xscale: float = 1.0, round_fn=None) -> np.ndarray:
    """Return a copy of x with near-tie rows re-drawn.  ``round_fn`` (e.g. a
    bf16 round-trip) is applied to re-drawn rows so the guard holds for the
    values the GPU will actually see."""
    x = np.array(x, dtype=np.float64, copy=True)
    o = restatement()
    base = o.derive_seed(layer_seed, "redraw")
    for attempt in range(64):
        gap, lmax = gaps(x, gate_w, cfg, phase, layer_seed)
        bad = np.nonzero(gap < rel_delta * lmax)[0]
        if bad.size == 0:
            return x
        for t in bad:
            row = uniform(o.derive_seed(base, int(t) * 1024 + attempt), x.shape[1], -xscale, xscale)
            x[t] = round_fn(row) if round_fn is not None else row
    raise RuntimeError("margin_guard did not converge")
