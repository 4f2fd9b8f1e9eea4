"""Host<->device copy bandwidth from pinned memory, per GPU, with all ranks
copying at once (torchrun) — the ceiling of bench.py's e2e leg."""
import os
import time

import torch
import torch.distributed as dist

rank = int(os.environ.get("RANK", 0))
world = int(os.environ.get("WORLD_SIZE", 1))
if world > 1:
    dist.init_process_group("gloo")
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
n = 64 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)),
                 ("d2h", lambda: h.copy_(d, non_blocking=True)),
                 ("both", None)]:
    for _ in range(3):
        if fn:
            fn()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.time()
    reps = 20
    for _ in range(reps):
        if fn:
            fn()
        else:
            with torch.cuda.stream(s1):
                d.copy_(h, non_blocking=True)
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.time() - t0
    gbs = n * reps / dt / 1e9 * (2 if fn is None else 1)
    print(f"rank {rank}/{world} {name}: {gbs:.1f} GB/s", flush=True)
