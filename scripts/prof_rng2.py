import ctypes as C, sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2109_10465_b200 import _lib
lib = _lib.load()
raw = torch.empty(8192 * 2048, dtype=torch.int64, device="cuda")
for n in (148 * 312, 148 * 312 * 8, 148 * 312 * 64, 8192 * 2048):
    for i in range(3):
        lib.moe_debug_mt64_device(4217090220841641567 + i, n, C.c_void_p(raw.data_ptr()))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(5):
        lib.moe_debug_mt64_device(4217090220841641567 + i, n, C.c_void_p(raw.data_ptr()))
    e1.record(); torch.cuda.synchronize()
    print(n, "ms per generation (incl. sync)", e0.elapsed_time(e1) / 5)
