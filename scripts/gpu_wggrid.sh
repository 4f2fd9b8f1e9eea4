cd $GRAFT_REPO_ROOT
./build/micro/tma_store_bw
for g in 148 128 120 112 96; do
MOE_B200_WG_BR=0 MOE_B200_WG_GRID=$g timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('grid=$g', round(l['ms_per_step'],4), {k:round(v,4) for k,v in l['stages_ms'].items() if 'wgrad' in k})"
done
