# A/B of bench.py command-line variants on one box: AB_ARGS0 / AB_ARGS1
cd $GRAFT_REPO_ROOT
for i in 1 2 3; do for v in 0 1; do
if [ $v = 0 ]; then A="$AB_ARGS0"; else A="$AB_ARGS1"; fi
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline $A 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('args=$v', round(l['value']/1e6,3), round(l['ms_per_step'],4), {k[:10]:round(v,4) for k,v in l['stages_ms'].items() if v>0.005})"
done; done
