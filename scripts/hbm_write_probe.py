"""Pure-write / pure-read / copy HBM bandwidth on one GPU (torch kernels),
to put the write-bound weight-gradient GEMMs in context."""
import torch
n = 4 << 30  # bytes
a = torch.empty(n // 2, dtype=torch.bfloat16, device="cuda")
b = torch.empty_like(a)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
def t(fn, nbytes, reps=10):
    fn(); torch.cuda.synchronize()
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9
print("write (fill)  GB/s", round(t(lambda: a.fill_(1.0), n)))
print("read  (sum)   GB/s", round(t(lambda: a.sum(), n)))
print("copy          GB/s", round(t(lambda: b.copy_(a), 2 * n)))
