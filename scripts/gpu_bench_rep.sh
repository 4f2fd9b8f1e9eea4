cd $GRAFT_REPO_ROOT
for a in "--steps 20 --warmup 5" "--steps 20 --warmup 5 --no-cpu-baseline" "--steps 30 --warmup 5 --no-cpu-baseline" "--steps 20 --warmup 5"; do
timeout 600 python bench.py $a 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$a', round(l['value']/1e6,3), round(l['ms_per_step'],4), round(l['e2e']['value']/1e6,3), {k[:10]:round(v,4) for k,v in l['stages_ms'].items() if not k.startswith('ffn')})"
done
