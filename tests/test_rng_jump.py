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
@pytest.mark.parametrize("count", [1, 311, 312, 5000, 2_000_003, 16_777_216])
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
