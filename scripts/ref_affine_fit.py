"""Cross-check of the reference arm's sampling.

The reference computes every capacity row of every expert, one expert after
another (routing.cpp:397-406), so config 3's fwd+bwd time on one rank is
  t(E=64, cap=128) = sum over 64 experts of the same (cap=128, d=2048,
  f=8192) expert work + the gate / assignment / combine (O(T d E), <1%)
  + the weight-gradient zero-fill, itself per expert.
bench.py --impl reference times exactly one expert's share (E'=1, cap=128,
128 tokens) as concurrent replicas.  This script checks that decomposition
against BASELINE.md §3a's method: the FULL 64-expert layer at two reduced
token counts (same d, f, E), an affine fit t = a + b R in padded rows
R = E * cap, extrapolated to T = 8192 (labelled extrapolated), next to 64x the
one-expert sample — all single-threaded on this host.

  python scripts/ref_affine_fit.py [--out profiles/r02_reference_fit.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402


def timed(T, E, d=2048, f=8192, seed=42):
    x, gw, w1, b1, w2, b2, dy = O.layer_inputs(T, d, f, E, seed=seed)
    cfg = O.make_cfg(num_experts=E, jitter_eps=0.01, balance_coeff=0.01)
    cap = O.restatement().capacity(T, cfg, O.TRAIN)
    t0 = time.perf_counter()
    secs = O.time_reference_layer(x, gw, w1, b1, w2, b2, cfg, O.TRAIN, 42, dy, 1)
    wall = time.perf_counter() - t0
    del x, w1, w2
    return dict(T=T, E=E, cap=cap, R=E * cap, secs=secs, wall=wall)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_reference_fit.json"))
    ap.add_argument("--tokens", type=int, nargs=2, default=[512, 1024])
    a = ap.parse_args()
    assert O.have_reference(), "oracle/_ref/libmoeforge_ref.so is required (make -C oracle ref)"
    one = timed(128, 1)
    print("one expert, cap 128:", one, flush=True)
    pts = []
    for T in a.tokens:
        p = timed(T, 64)
        print("E=64:", p, flush=True)
        pts.append(p)
    (r0, t0), (r1, t1) = [(p["R"], p["secs"]) for p in pts]
    b = (t1 - t0) / (r1 - r0)
    av = t0 - b * r0
    R = 64 * 128
    pred = av + b * R
    out = dict(host_cores=os.cpu_count(), one_expert=one, full_layer_points=pts,
               fit=dict(a_s=av, b_s_per_row=b, R_c3=R, t_c3_extrapolated_s=pred,
                        tokens_per_s_extrapolated=8192 / pred),
               decomposition=dict(t_c3_64x_one_expert_s=64 * one["secs"],
                                  tokens_per_s=8192 / (64 * one["secs"])),
               ratio_fit_over_decomposition=pred / (64 * one["secs"]),
               note="single-threaded reference (oracle/_ref) on the GPU box host; the fit is "
                    "extrapolated from T=%d/%d" % tuple(a.tokens))
    print(json.dumps(out, indent=1))
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
