"""Per-phase timeline of the device jitter generator (debug build switch
MOE_B200_RNG_TIMING=1) plus CUDA-event timing of the whole launch."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_10465_b200 import _lib  # noqa: E402

L = _lib.load()
count = int(sys.argv[1]) if len(sys.argv) > 1 else 8192 * 2048
out = torch.empty(count, dtype=torch.float32, device="cuda")
for _ in range(3):
    assert L.moe_debug_jitter_device(12345, count, 0.01, C.c_void_p(out.data_ptr())) == 0
if not os.environ.get("MOE_B200_RNG_TIMING"):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        L.moe_debug_jitter_device(12345, count, 0.01, C.c_void_p(out.data_ptr()))
    e1.record()
    torch.cuda.synchronize()
    print(f"jitter {count} values: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us/call (incl. sync)")
