cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "bf16 or prefetch or fused or pdl" 2>&1 | tail -3
python scripts/micro/gate_probe.py 2>&1 | grep -v Warning | head -3
for s in 10 12 14; do for hold in 0 1; do
  MOE_B200_PF_SMS=$s MOE_B200_PF_HOLD=$hold timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('sms=$s hold=$hold', round(l['value']/1e6,3), round(l['ms_per_step'],4), {k:v for k,v in l['stages_ms'].items() if k in ('gate_fused','ffn1_fwd','ffn2_dgrad','ffn2_wgrad','ffn1_wgrad')})"
done; done
