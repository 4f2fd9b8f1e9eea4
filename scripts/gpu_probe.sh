# fused-gate timing probes + jitter prefetch variants (gpurun)
cd $GRAFT_REPO_ROOT
python scripts/micro/gate_probe.py 2>&1 | grep -v Warning
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k prefetch 2>&1 | tail -2
for s in 8 16; do
  MOE_B200_PF_SMS=$s timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --prefetch 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('prefetch sms=$s', round(l['value']/1e6,3), round(l['ms_per_step'],4), {k:v for k,v in l['stages_ms'].items() if 'ffn' in k or 'jit' in k})"
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('no prefetch', round(l['value']/1e6,3), round(l['ms_per_step'],4), {k:v for k,v in l['stages_ms'].items() if 'ffn' in k or 'jit' in k})"
