"""Build libmoe_b200.so in-tree for sm_100a (``python -m paper_2109_10465_b200.build``)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def build(jobs: int = 8, verbose: bool = False) -> str:
    cmd = ["make", "-C", os.path.join(HERE, "csrc"), f"-j{jobs}"]
    r = subprocess.run(cmd, capture_output=not verbose, text=True)
    if r.returncode != 0:
        sys.stderr.write((r.stdout or "") + (r.stderr or ""))
        raise RuntimeError("libmoe_b200.so build failed")
    return os.path.join(HERE, "libmoe_b200.so")


if __name__ == "__main__":
    print(build(verbose=True))
