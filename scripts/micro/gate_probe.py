"""Time the forward stages of a config-3 bf16 layer under the fused-gate timing
probes (MOE_B200_GATE_PROBE: 1 = no 3xTF32 split math, 2 = no MMA, 4 = no
last-CTA finalize; results are wrong under probes — timing only)."""
import os
import subprocess
import sys

CODE = r'''
import torch, sys, os
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"] if "GRAFT_REPO_ROOT" in os.environ else ".")
import paper_2109_10465_b200 as M
T, d, f, E = 8192, 2048, 8192, 64
g = torch.Generator(device="cuda").manual_seed(1)
L = M.MoeLayer(M.RouterConfig(num_experts=E), T, d, f, torch.bfloat16)
r = lambda *s: (torch.rand(*s, device="cuda", generator=g) * 2 - 1)
p = M.MoeLayerParams(r(d, E) * 0.05, (r(E, d, f) * 0.02).bfloat16(), r(E, f) * 0.01,
                     (r(E, f, d) * 0.02).bfloat16(), r(E, d) * 0.01)
x = r(T, d).bfloat16()
for i in range(5):
    L.forward(x, p, M.Phase.TRAIN, 42 + i, decision=False, check=False)
torch.cuda.synchronize()
L.handle.profile(True)
for i in range(20):
    L.forward(x, p, M.Phase.TRAIN, 42 + i, decision=False, check=False)
st = L.handle.profile_read()
print(os.environ.get("MOE_B200_GATE_PROBE", "0"), {k: round(v[0] / v[1] * 1e3, 1) for k, v in st.items()})
'''
for probe in ["0", "1", "2", "3", "4", "7"]:
    env = dict(os.environ, MOE_B200_GATE_PROBE=probe)
    subprocess.run([sys.executable, "-c", CODE], env=env)
