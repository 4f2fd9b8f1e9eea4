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


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_ep_two_ranks_matches_per_rank_composition(mode):
    n = ngpus()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    w = min(n, 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={w}",
           "--master-addr", "127.0.0.1", "--master-port", str(29511 + (mode == "bf16")),
           os.path.join(ROOT, "tests", "ep_check.py"), mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0 and "EP_OK" in r.stdout
