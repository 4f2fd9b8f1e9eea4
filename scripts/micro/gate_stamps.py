"""Phase timeline of the fused gate kernel (MOE_B200_GATE_PROBE=8): per-CTA
%globaltimer stamps, relative to the earliest CTA start (us)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
os.environ["MOE_B200_GATE_PROBE"] = "8"
import paper_2109_10465_b200 as M  # noqa: E402
from paper_2109_10465_b200 import _lib  # noqa: E402

T, d, f, E = 8192, 2048, 256, 64
g = torch.Generator(device="cuda").manual_seed(1)
L = M.MoeLayer(M.RouterConfig(num_experts=E), T, d, f, torch.bfloat16)
r = lambda *s: (torch.rand(*s, device="cuda", generator=g) * 2 - 1)  # noqa: E731
p = M.MoeLayerParams(r(d, E) * 0.05, (r(E, d, f) * 0.02).bfloat16(), r(E, f) * 0.01,
                     (r(E, f, d) * 0.02).bfloat16(), r(E, d) * 0.01)
x = r(T, d).bfloat16()
for i in range(4):
    L.forward(x, p, M.Phase.TRAIN, 42 + i, decision=False, check=False)
torch.cuda.synchronize()
ncta = 2 * T // 128
buf = np.zeros(ncta * 8, np.uint64)
n = C.c_int()
_lib.load().moe_debug_gate_stamps(buf.ctypes.data_as(C.c_void_p), ncta, C.byref(n))
s = buf.reshape(ncta, 8).astype(np.float64)
t0 = s[:, 0].min()
names = ["start", "after pdl_wait", "acc ready", "before cluster", "after cluster", "routing done"]
for i, nm in enumerate(names):
    v = (s[:, i] - t0) / 1e3
    print(f"{nm:16s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f} us")
