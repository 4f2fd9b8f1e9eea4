import ctypes as C, torch, sys
sys.path.insert(0, '.')
from paper_2109_10465_b200 import _lib as L
lib = L.load()
p = lambda t: C.c_void_p(t.data_ptr())
T, d, E = 256, 256, 64
x = torch.ones(T, d, device="cuda", dtype=torch.bfloat16)
wg = torch.ones(d, E, device="cuda")
out = torch.full((1, T, E), -7.0, device="cuda")
print("st", lib.moe_debug_gate_tc_logits(p(x), None, p(wg), p(out), T, d, E, 1))
print(out[0, :3, :8], out.abs().sum())
dL = torch.ones(T, E, device="cuda")
part = torch.full((1, d, E), -7.0, device="cuda")
print("st", lib.moe_debug_gate_tc_dw(p(x), p(torch.ones(T, d, device="cuda")), p(dL), p(part), T, d, E, 1))
print(part[0, :3, :8])
