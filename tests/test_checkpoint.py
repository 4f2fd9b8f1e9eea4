"""§8(f) row 2: checkpoint -> device weight layout.  Checkpoints are written
and pruned by the reference's own checkpoint.cpp / surgery.cpp (oracle/_ref);
the loader must read them with the reference's checks (version, blob size,
CRC32, record length) and prune identically (surgery.cpp:135-212)."""
import json
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.skipif(not O.have_reference(), reason="reference not built")


@pytest.fixture(scope="module")
def ckpt_dir(tmp_path_factory):
    d = tmp_path_factory.mktemp("ckpt") / "toy"
    O.ref_save_toy_checkpoint(d)
    return d


def test_load_reference_checkpoint(ckpt_dir):
    from paper_2109_10465_b200.checkpoint import load_checkpoint, moe_layer_prefixes
    ck = load_checkpoint(ckpt_dir)
    man = json.load(open(os.path.join(ckpt_dir, "manifest.json")))
    assert [r.name for r in ck.tensors] == [t["name"] for t in man["tensors"]]
    assert ck.num_moe_layers() == 2
    assert moe_layer_prefixes(ck) == ["enc.1", "dec.1"]
    g = ck.at("enc.1.moe.gate")
    assert g.shape == [64, 8] and g.role == "gate" and g.layer == 0
    w = ck.at("dec.1.moe.expert3.w2")
    assert w.shape == [128, 64] and w.expert == 3 and w.layer == 1


def test_checkpoint_integrity_errors(ckpt_dir, tmp_path):
    import shutil
    from paper_2109_10465_b200.checkpoint import CheckpointError, load_checkpoint
    bad = tmp_path / "bad"
    shutil.copytree(ckpt_dir, bad)
    blob = bad / "tensors.bin"
    raw = bytearray(blob.read_bytes())
    raw[100] ^= 0x01
    blob.write_bytes(bytes(raw))
    with pytest.raises(CheckpointError, match="checksum failure"):
        load_checkpoint(bad)
    blob.write_bytes(bytes(raw[:-8]))
    with pytest.raises(CheckpointError, match="blob truncated or oversized"):
        load_checkpoint(bad)
    m = json.load(open(bad / "manifest.json"))
    m["version"] = "moe-forge-ckpt/0"
    json.dump(m, open(bad / "manifest.json", "w"))
    with pytest.raises(CheckpointError, match="version mismatch"):
        load_checkpoint(bad)


@pytest.mark.parametrize("strategy,k", [("top_utilization", 3), ("random", 4), ("top_utilization", 8)])
def test_prune_matches_reference(ckpt_dir, tmp_path, strategy, k):
    from paper_2109_10465_b200.checkpoint import load_checkpoint, prune_experts
    counts = [[5, 9, 9, 1, 0, 7, 3, 9], [0, 0, 2, 2, 8, 1, 1, 6]]  # ties break to the lower index
    O.ref_prune_checkpoint(ckpt_dir, tmp_path / "p", k, strategy, counts if strategy == "top_utilization" else None,
                           seed=11)
    ref = load_checkpoint(tmp_path / "p")
    ours = prune_experts(load_checkpoint(ckpt_dir), k, strategy, counts, seed=11)
    assert ours.arch == ref.arch
    assert [r.name for r in ours.tensors] == [r.name for r in ref.tensors]
    for a, b in zip(ours.tensors, ref.tensors):
        assert a.shape == b.shape and np.array_equal(a.data, b.data), a.name


def _bf16_rne(a):
    """Correctly rounded f64 -> bf16 (round half to even), as exact float32
    values.  torch's CPU f64 -> bf16 cast goes through float32 and can double
    round, so it is not the reference for a one-step device conversion."""
    m, e = np.frexp(np.asarray(a, np.float64))
    return np.ldexp(np.rint(m * 256.0), e - 8).astype(np.float32)


@pytest.mark.gpu
def test_pack_to_device_layout(ckpt_dir):
    import torch
    import paper_2109_10465_b200 as M
    from paper_2109_10465_b200.checkpoint import load_checkpoint, moe_layer_params
    ck = load_checkpoint(ckpt_dir)
    for ordinal, prefix in enumerate(["enc.1", "dec.1"]):
        p = moe_layer_params(ck, ordinal, torch.bfloat16)
        w1 = np.stack([ck.at(f"{prefix}.moe.expert{e}.w1").data.reshape(64, 128) for e in range(8)])
        assert torch.equal(p.w1.cpu(), torch.from_numpy(_bf16_rne(w1)).to(torch.bfloat16))
        w2 = np.stack([ck.at(f"{prefix}.moe.expert{e}.w2").data.reshape(128, 64) for e in range(8)])
        assert torch.equal(p.w2.cpu(), torch.from_numpy(_bf16_rne(w2)).to(torch.bfloat16))
        g = ck.at(f"{prefix}.moe.gate").data.reshape(64, 8)
        assert torch.equal(p.gate_w.cpu(), torch.from_numpy(g).float())
        # the packed layer runs
        layer = M.MoeLayer(M.RouterConfig(num_experts=8), 128, 64, 128, torch.bfloat16)
        x = torch.rand(128, 64, device="cuda").to(torch.bfloat16)
        y, aux, dec = layer.forward(x, p, M.Phase.EVAL, 1)
        assert torch.isfinite(y.float()).all()
    # expert-parallel shard: experts [4, 8) of layer 0
    sh = moe_layer_params(ck, 0, torch.float32, experts=range(4, 8))
    w1 = np.stack([ck.at(f"enc.1.moe.expert{e}.w1").data.reshape(64, 128) for e in range(4, 8)])
    assert torch.equal(sh.w1.cpu(), torch.from_numpy(w1).float())
