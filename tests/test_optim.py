"""§8(f) row 4: the expert optimizer step.  CPU: the oracle's restatement of
AdamOptimizer (optim.cpp:21-57) against the reference's own class
(oracle/_ref).  GPU: the device Adam (optim.cu) against the restatement."""
import numpy as np
import pytest

import oracle as O


def _case(seed, sizes, steps):
    rng = np.random.default_rng(seed)
    th = [rng.standard_normal(n) for n in sizes]
    gs = [[rng.standard_normal(n) * (0.5 + s) for n in sizes] for s in range(steps)]
    lrs = [1e-3 * (1 + s % 3) for s in range(steps)]
    return th, gs, lrs


@pytest.mark.skipif(not O.have_reference(), reason="reference not built")
@pytest.mark.parametrize("clip", [0.0, 1.0, 50.0])
def test_adam_restatement_matches_reference(clip):
    th, gs, lrs = _case(1, [5, 64, 300], 5)
    a = O.adam_restated(th, gs, lrs, clip=clip)
    b = O.adam_reference(th, gs, lrs, clip=clip)
    for x, y in zip(a[0] + a[1] + a[2], b[0] + b[1] + b[2]):
        assert np.array_equal(x, y)


def test_adam_rejects_nonpositive_lr():
    with pytest.raises(ValueError):
        O.adam_restated([np.zeros(3)], [[np.zeros(3)]], [0.0])


@pytest.mark.gpu
@pytest.mark.parametrize("clip,gdt", [(0.0, "fp32"), (1.0, "fp32"), (5.0, "bf16")])
def test_device_adam_matches_restatement(clip, gdt):
    import torch
    from paper_2109_10465_b200.optim import Adam
    sizes = [1000, 4097, 70000]
    th, gs, lrs = _case(2, sizes, 4)
    tdt = torch.float32 if gdt == "fp32" else torch.bfloat16
    # the device sees fp32 masters and fp32 / bf16 gradients: feed the oracle those values
    th32 = [np.asarray(t, np.float32).astype(np.float64) for t in th]
    gdev = [[torch.from_numpy(np.asarray(g, np.float32)).to("cuda", tdt) for g in gl] for gl in gs]
    g64 = [[g.float().cpu().numpy().astype(np.float64) for g in gl] for gl in gdev]
    ref_th, ref_m, ref_v = O.adam_restated(th32, g64, lrs, clip=clip)
    params = [torch.from_numpy(t.astype(np.float32)).cuda() for t in th32]
    shadows = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for n in sizes]
    opt = Adam(params, shadows=shadows)
    for s in range(len(lrs)):
        opt.step(gdev[s], lrs[s], clip_norm=clip)
    torch.cuda.synchronize()
    for i in range(len(sizes)):
        p = params[i].cpu().numpy().astype(np.float64)
        # fp32 storage of theta/m/v between steps: ~1e-7 relative per step
        assert np.max(np.abs(p - ref_th[i])) <= 1e-6 * max(1.0, np.max(np.abs(ref_th[i])))
        assert np.max(np.abs(opt.m[i].cpu().numpy() - ref_m[i])) <= 1e-6 * max(1e-3, np.max(np.abs(ref_m[i])))
        assert torch.equal(shadows[i], params[i].to(torch.bfloat16))
    assert opt.step_count == len(lrs)
