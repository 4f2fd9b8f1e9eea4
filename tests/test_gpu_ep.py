"""Expert parallelism, one process per rank (tests/ep_check.py under torchrun).

Two families:
* ranks on separate GPUs (skip on a 1-GPU box): NCCL-bootstrapped, every
  transport (NVLink peer stores in the GEMM epilogues + peer copies + flag
  barrier; the copy-pass, NCCL-barrier and NCCL send/recv fallbacks), plus the
  config-3-shaped case (E=64, d=2048, f=8192);
* two ranks SHARING one GPU (runs on the 1-GPU box): bootstrapped without
  NCCL (moe_ep_export / moe_ep_import over gloo), the same NVLink-path code —
  IPC-mapped receive buffers, peer-store GEMM epilogues, the device flag
  barrier — exercised against the per-rank oracle composition, including the
  config-3 widths and the UniformShapeError contract.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpus():
    import torch
    return torch.cuda.device_count()


def run_ep(world, args, env=None, port=29511, timeout=900):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "ep_check.py"), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT,
                       env=dict(os.environ, **(env or {})))
    print(r.stdout[-4000:], r.stderr[-3000:])
    assert r.returncode == 0 and "EP_OK" in r.stdout
    return r.stdout


# transports: default = NVLink peer stores (GEMM epilogues + peer copies, flag
# barrier); the fallbacks: copy pass instead of the epilogue stores, NCCL
# all-reduce barrier, NCCL send/recv for everything
TRANSPORTS = {"default": {}, "copy": {"MOE_B200_PEER_EPI": "0"},
              "nccl_barrier": {"MOE_B200_EP_BARRIER": "nccl"}, "nccl": {"MOE_B200_EP_TRANSPORT": "nccl"}}


@pytest.mark.parametrize("mode,transport", [("fp32", "default"), ("bf16", "default"), ("bf16", "copy"),
                                            ("bf16", "nccl_barrier"), ("bf16", "nccl")])
def test_ep_multi_gpu_matches_per_rank_composition(mode, transport):
    n = ngpus()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    port = 29511 + 2 * list(TRANSPORTS).index(transport) + (mode == "bf16")
    run_ep(min(n, 4), [mode], TRANSPORTS[transport], port)


@pytest.mark.parametrize("transport", ["default", "nccl"])
def test_ep_multi_gpu_c3_shape(transport):
    n = ngpus()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    run_ep(min(n, 4), ["bf16", "--shape", "c3"], TRANSPORTS[transport], 29531 + (transport == "nccl"))


def test_ep_multi_gpu_uniform_shape_error():
    n = ngpus()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    run_ep(min(n, 4), ["bf16", "--uneven"], port=29535)


# ---- two ranks on one GPU (NCCL-free bootstrap) ---------------------------------
@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_ep_shared_gpu_matches_per_rank_composition(mode):
    run_ep(2, [mode, "--bootstrap", "ipc", "--same-gpu"], port=29541 + (mode == "bf16"))


def test_ep_shared_gpu_copy_transport():
    run_ep(2, ["bf16", "--bootstrap", "ipc", "--same-gpu"], TRANSPORTS["copy"], port=29543)


def test_ep_shared_gpu_c3_shape():
    run_ep(2, ["bf16", "--shape", "c3", "--bootstrap", "ipc", "--same-gpu"], port=29545)


def test_ep_shared_gpu_uniform_shape_error():
    out = run_ep(2, ["bf16", "--bootstrap", "ipc", "--same-gpu", "--uneven"], port=29547)
    assert out.count("UniformShapeError") == 2
