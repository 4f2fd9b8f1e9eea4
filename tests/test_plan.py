"""The capacity check: the ZeRO-2 / EP memory planner
of libmoe_b200.so (plan.cpp) against the reference's own memory_per_gpu /
max_model_size (oracle/_ref, parallel.cpp:18-115) over a grid of plans, and
the reference's known answers (test_parallel.cpp:38-140).  CPU only."""
import ctypes as C
import itertools

import numpy as np
import pytest

import oracle as O
from paper_2109_10465_b200 import plan as P
from paper_2109_10465_b200.routing import ConfigError


class _RefPlan(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("world_size", "expert_parallel", "model_parallel", "zero_stage",
                                         "offload")]


def _ref():
    if not O.have_reference():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    lib = O.reference().lib
    lib.ref_memory_per_gpu.argtypes = [C.POINTER(_RefPlan), C.c_double, C.c_double, C.POINTER(C.c_double)]
    lib.ref_max_model_size.argtypes = [C.POINTER(_RefPlan), C.c_double, C.c_double, C.c_double,
                                       C.POINTER(C.c_int64), C.POINTER(C.c_double)]
    return lib


def plans():
    for N, ep, mp, z, off in itertools.product([1, 2, 4, 8, 16], [1, 2, 4, 8], [1, 2], [0, 1, 2], [0, 1]):
        yield P.ParallelPlan(N, ep, mp, z, bool(off))


def test_memory_per_gpu_matches_reference_grid():
    lib = _ref()
    n_ok = n_err = 0
    for p in plans():
        for ne, ex in ((1e9, 0.0), (7e8, 3e8), (1_179_648, 9_669_574_656), (6e8, 4e9)):
            out = (C.c_double * 7)()
            st = lib.ref_memory_per_gpu(C.byref(_RefPlan(p.world_size, p.expert_parallel, p.model_parallel,
                                                         p.zero_stage, int(p.offload))), ne, ex, out)
            if st:
                with pytest.raises(ConfigError):
                    P.memory_per_gpu(p, ne, ex)
                n_err += 1
                continue
            e = P.memory_per_gpu(p, ne, ex)
            mine = [e.nonexpert_params, e.expert_params, e.nonexpert_grads, e.expert_grads,
                    e.nonexpert_optim, e.expert_optim, e.gpu_total()]
            assert np.array_equal(np.array(mine), np.array(out[:])), (p, ne, ex)
            n_ok += 1
    assert n_ok > 100 and n_err > 50


def test_max_model_size_matches_reference():
    lib = _ref()
    for p in plans():
        rp = _RefPlan(p.world_size, p.expert_parallel, p.model_parallel, p.zero_stage, int(p.offload))
        for budget, base, per in ((1.6e9, 50e6, 10e6), (180e9, 1e9, 268_451_840), (40e9, 15e9, 5e8)):
            n, tot = C.c_int64(), C.c_double()
            st = lib.ref_max_model_size(C.byref(rp), budget, base, per, C.byref(n), C.byref(tot))
            if st:
                with pytest.raises(ConfigError):
                    P.max_model_size(p, budget, base, per)
                continue
            assert P.max_model_size(p, budget, base, per) == (n.value, tot.value)


def test_reference_known_answers():
    # test_parallel.cpp:38-140
    ok = P.ParallelPlan(8, 4, 2, 2)
    ok.validate()
    for bad in (P.ParallelPlan(8, 3, 2, 2), P.ParallelPlan(8, 4, 2, 1), P.ParallelPlan(8, 4, 3, 2),
                P.ParallelPlan(8, 8, 2, 2)):
        with pytest.raises(ConfigError):
            bad.validate()
    e = P.memory_per_gpu(P.ParallelPlan(), 1e9, 0.0)
    assert e.gpu_total() == pytest.approx(16e9, rel=1e-12) and e.cpu_total() == 0.0
    assert P.memory_per_gpu(P.ParallelPlan(), 7e8, 3e8).optimizer_grad_share() == pytest.approx(0.875, rel=1e-12)
    e = P.memory_per_gpu(P.ParallelPlan(offload=True), 1e9, 0.0)
    assert e.gpu_total() == pytest.approx(2e9, rel=1e-12) and e.cpu_total() == pytest.approx(14e9, rel=1e-12)
    n0, t0 = P.max_model_size(P.ParallelPlan(), 1.6e9, 10e6, 1e6)
    n1, t1 = P.max_model_size(P.ParallelPlan(offload=True), 1.6e9, 10e6, 1e6)
    assert t0 == pytest.approx(100e6, rel=1e-12) and t1 == pytest.approx(800e6, rel=1e-12)
    with pytest.raises(ConfigError):
        P.max_model_size(P.ParallelPlan(), 1e6, 50e6, 10e6)   # base alone exceeds the budget


def test_capacity_check_config4():
    """The paper's 10B-class stack (config 4: 18 MoE layers, d=1024, f=4096,
    E=64; 10,279,540,736 params per the oracle's param_count) at 8 GPUs with
    EP=8 and ZeRO-2 needs ~19.3 GB per 180 GB B200 for its MoE-layer state; on
    one GPU it needs 165 GB, and twice the stack does not fit."""
    ne1, ex1 = P.layer_params(1024, 4096, 64)
    ne, ex = 18 * ne1, 18 * ex1
    fit = P.capacity_check(P.ParallelPlan(8, 8, 1, 2), ne, ex, hbm_bytes=180e9)
    assert 19e9 < fit["total_bytes"] < 20e9
    one = P.capacity_check(P.ParallelPlan(1, 1, 1, 0), ne, ex, hbm_bytes=180e9)
    assert one["total_bytes"] == pytest.approx(16.0 * (ne + ex))
    with pytest.raises(ConfigError):
        P.capacity_check(P.ParallelPlan(1, 1, 1, 0), 2 * ne, 2 * ex, hbm_bytes=180e9)
