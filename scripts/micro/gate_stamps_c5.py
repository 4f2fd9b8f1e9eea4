"""Phase timeline of the fused gate on a config-5 shape (eval, no jitter):
MOE_B200_GATE_PROBE=8 %globaltimer stamps per CTA, relative to the earliest
CTA start (us).  Usage: gate_stamps_c5.py [E] [T] [d] [train]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
os.environ["MOE_B200_GATE_PROBE"] = os.environ.get("GATE_PROBE", "8")
import paper_2109_10465_b200 as M  # noqa: E402
from paper_2109_10465_b200 import _lib  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 16
T = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
d = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
f = 256
train = len(sys.argv) > 4 and sys.argv[4] != "0"
g = torch.Generator(device="cuda").manual_seed(1)
L = M.MoeLayer(M.RouterConfig(num_experts=E), T, d, f, torch.bfloat16)
r = lambda *s: (torch.rand(*s, device="cuda", generator=g) * 2 - 1)  # noqa: E731
p = M.MoeLayerParams(r(d, E) * 0.05, (r(E, d, f) * 0.02).bfloat16(), r(E, f) * 0.01,
                     (r(E, f, d) * 0.02).bfloat16(), r(E, d) * 0.01)
x = r(T, d).bfloat16()
for i in range(4):
    L.forward(x, p, M.Phase.TRAIN if train else M.Phase.EVAL, 42 + i, decision=False, check=False)
torch.cuda.synchronize()
tiles = (T + 127) // 128
sm2 = E <= 16 and not train and os.environ.get("MOE_B200_GATE_SM2", "1") != "0"
ncta = tiles * (1 if tiles > (148 if sm2 else 74) else 2)
buf = np.zeros(ncta * 8, np.uint64)
n = C.c_int()
_lib.load().moe_debug_gate_stamps(buf.ctypes.data_as(C.c_void_p), ncta, C.byref(n))
s = buf.reshape(ncta, 8).astype(np.float64)
t0 = s[:, 0].min()
print(f"E={E} T={T} d={d} CTAs={ncta}  kernel span {(s[:, 5].max() - t0) / 1e3:.1f} us")
names = ["start", "after pdl_wait", "acc ready", "before cluster", "after cluster", "routing done"]
for i, nm in enumerate(names):
    v = (s[:, i] - t0) / 1e3
    print(f"{nm:16s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f} us")
dur = (s[:, 5] - s[:, 0]) / 1e3
loop = (s[:, 2] - s[:, 1]) / 1e3
print(f"per CTA: total med {np.median(dur):.2f} us, main loop med {np.median(loop):.2f} us")
