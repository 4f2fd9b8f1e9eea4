cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "bf16 or prefetch or fused or pdl or parity or ep_shared" 2>&1 | tail -3
for s in 6 8 10 12; do
  MOE_B200_PF_SMS=$s timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('prefetch sms=$s', round(l['value']/1e6,3), round(l['ms_per_step'],4), l['stages_ms'])"
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-prefetch 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('no prefetch', round(l['value']/1e6,3), round(l['ms_per_step'],4), l['stages_ms'])"
