"""Per-stage timeline of the fused gate's main loop (MOE_B200_GATE_PROBE=16, on a build
with -DMOE_GATE_TIMELINE, e.g. scripts/build_variants.sh gate_fused.cu tl:"-DMOE_GATE_TIMELINE"
and MOE_B200_LIB pointing at it):
for CTA 0, when the producer issued each raw stage, when the transform saw it
land and finished it, and when the MMA issued its second step (us from the
first issue).  Usage: gate_timeline.py [E] [T] [d] [train]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
os.environ["MOE_B200_GATE_PROBE"] = os.environ.get("GATE_PROBE", "16")
import paper_2109_10465_b200 as M  # noqa: E402
from paper_2109_10465_b200 import _lib  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 64
T = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
d = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
train = (sys.argv[4] != "0") if len(sys.argv) > 4 else True
f = 256
g = torch.Generator(device="cuda").manual_seed(1)
L = M.MoeLayer(M.RouterConfig(num_experts=E), T, d, f, torch.bfloat16)
r = lambda *s: (torch.rand(*s, device="cuda", generator=g) * 2 - 1)  # noqa: E731
p = M.MoeLayerParams(r(d, E) * 0.05, (r(E, d, f) * 0.02).bfloat16(), r(E, f) * 0.01,
                     (r(E, f, d) * 0.02).bfloat16(), r(E, d) * 0.01)
x = r(T, d).bfloat16()
ph = M.Phase.TRAIN if train else M.Phase.EVAL
for i in range(4):
    L.forward(x, p, ph, 42 + i, decision=False, check=False)
torch.cuda.synchronize()
buf = np.zeros(8 * 64, np.uint64)
n = C.c_int()
_lib.load().moe_debug_gate_stamps(buf.ctypes.data_as(C.c_void_p), 64, C.byref(n))
tl = buf.reshape(8, 64).astype(np.float64)
for cta in (0, 1):
    t0 = tl[cta, 0]
    print(f"CTA {cta}: stage  issue  landed  done  mma(us)")
    for s in range(16):
        row = [(tl[cta, k * 16 + s] - t0) / 1e3 for k in range(4)]
        print(f"  {s:2d}   " + "  ".join(f"{v:6.2f}" for v in row))
