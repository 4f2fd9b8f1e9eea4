cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "${PYTEST_K:-fused or c3_full or bf16_tcgen05_vs_oracle}" 2>&1 | tail -2
python scripts/micro/gate_stamps.py 2>&1 | tail -6
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(l['value']/1e6,3), round(l['ms_per_step'],4), l['stages_ms'])"
