"""Expert parallelism over NCCL on >= 2 GPUs (skips on a 1-GPU box).
Runs tests/ep_check.py under torchrun (one process per GPU)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpus():
    import torch
    return torch.cuda.device_count()


# transports: default = NVLink peer stores (GEMM epilogues + peer copies, flag
# barrier); the fallbacks: copy pass instead of the epilogue stores, NCCL
# all-reduce barrier, NCCL send/recv for everything
TRANSPORTS = {"default": {}, "copy": {"MOE_B200_PEER_EPI": "0"},
              "nccl_barrier": {"MOE_B200_EP_BARRIER": "nccl"}, "nccl": {"MOE_B200_EP_TRANSPORT": "nccl"}}


@pytest.mark.parametrize("mode,transport", [("fp32", "default"), ("bf16", "default"), ("bf16", "copy"),
                                            ("bf16", "nccl_barrier"), ("bf16", "nccl")])
def test_ep_two_ranks_matches_per_rank_composition(mode, transport):
    n = ngpus()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    w = min(n, 4)
    port = 29511 + 2 * list(TRANSPORTS).index(transport) + (mode == "bf16")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={w}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "ep_check.py"), mode]
    env = dict(os.environ, **TRANSPORTS[transport])
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0 and "EP_OK" in r.stdout
