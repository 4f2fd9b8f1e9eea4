"""The device jitter generator reproduces the reference's mt19937_64 stream
(rng.cpp:36-43, routing.cpp:62-70) through polynomial jump-ahead.  CPU tests
pin the host half (characteristic polynomial + jump polynomials) against the
oracle's sequential stream; the GPU test pins the device kernels."""
import ctypes as C

import numpy as np
import pytest

import oracle as O


def _chunk_host(seed, J, c, n):
    from paper_2109_10465_b200 import _lib
    out = np.empty(n, np.uint64)
    st = _lib.load().moe_debug_mt64_chunk_host(seed, J, c, n, out.ctypes.data_as(C.c_void_p))
    assert st == 0
    return out


@pytest.mark.parametrize("seed,J,c,n", [(5489, 1000, 0, 400), (42, 1000, 3, 700),
                                        (O.restatement().derive_seed(42, "jitter"), 113511, 2, 640)])
def test_jump_ahead_host_matches_sequential_stream(seed, J, c, n):
    got = _chunk_host(seed, J, c, n)
    ref = O.restatement().mt64(seed, n, skip=c * J)
    assert np.array_equal(got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("count", [1, 311, 312, 313, 4097, 5000, 606_209, 2_000_003, 16_777_216])
def test_device_stream_matches_reference(count):
    import torch
    from paper_2109_10465_b200 import _lib
    seed = O.restatement().derive_seed(42, "jitter")
    out = torch.empty(count, dtype=torch.int64, device="cuda")
    assert _lib.load().moe_debug_mt64_device(seed, count, C.c_void_p(out.data_ptr())) == 0
    got = out.cpu().numpy().view(np.uint64)
    ref = O.restatement().mt64(seed, count)
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, (bad[:5], count)


@pytest.mark.gpu
@pytest.mark.parametrize("count,eps", [(5000, 0.01), (16_777_216, 0.01), (1_000_003, 0.25)])
def test_device_jitter_values_bit_exact(count, eps):
    """noise = (float)(lo + (hi - lo) * ((x >> 11) * 2^-53)) with the f64
    arithmetic of rng.cpp:36-43 (no fused multiply-add), then rounded to fp32."""
    import torch
    from paper_2109_10465_b200 import _lib
    seed = O.restatement().derive_seed(7, "jitter")
    out = torch.empty(count, dtype=torch.float32, device="cuda")
    assert _lib.load().moe_debug_jitter_device(seed, count, eps, C.c_void_p(out.data_ptr())) == 0
    raw = O.restatement().mt64(seed, count)
    lo, hi = 1.0 - eps, 1.0 + eps
    u = (raw >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    ref = (lo + (hi - lo) * u).astype(np.float32)
    got = out.cpu().numpy()
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
