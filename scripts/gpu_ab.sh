# A/B of an env toggle on one box: AB_VAR=NAME (values 0 / 1), optional PYTEST_K
cd $GRAFT_REPO_ROOT
if [ -n "$PYTEST_K" ]; then timeout 900 python -m pytest tests -m gpu -q -x -k "$PYTEST_K" 2>&1 | tail -2; fi
for i in 1 2 3; do for v in 0 1; do
env $AB_VAR=$v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$AB_VAR=$v', round(l['value']/1e6,3), round(l['ms_per_step'],4), {k[:10]:round(v,4) for k,v in l['stages_ms'].items() if v>0.005})"
done; done
