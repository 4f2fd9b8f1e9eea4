#!/bin/bash
# e2e leg A/B: dx + aux read back every step vs the aux loss only, plus the pinned-copy rates.
cd $GRAFT_REPO_ROOT
for i in 1 2; do for rb in dx aux; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-readback $rb 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$rb', round(l['value']/1e6,3), round(l['ms_per_step'],4), 'e2e', round(l['e2e']['value']/1e6,3), round(l['e2e']['ms_per_step'],4))"
done; done
python - <<'PY'
import torch, time
n = 8192 * 2048
a = torch.empty(n, dtype=torch.bfloat16).pin_memory(); b = torch.empty(n, dtype=torch.bfloat16, device="cuda")
c = torch.empty(n, dtype=torch.bfloat16).pin_memory(); e = torch.empty(n, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for mode in ("h2d", "d2h", "both"):
    torch.cuda.synchronize(); t = time.time()
    for _ in range(20):
        if mode in ("h2d", "both"):
            with torch.cuda.stream(s1): b.copy_(a, non_blocking=True)
        if mode in ("d2h", "both"):
            with torch.cuda.stream(s2): c.copy_(e, non_blocking=True)
    torch.cuda.synchronize(); dt = (time.time() - t) / 20
    print(mode, round(n * 2 / dt / 1e9, 1), "GB/s per direction")
PY
