# Development GPU session: focused tests, bench, launch list and one full ncu capture.
# PYTEST_K selects tests; NCU_KERNEL the kernel regex to capture (default: the fused gate).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rA ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/dev_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/dev_pytest.log | tail -15
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/dev_bench.json 2> gpurun_out/dev_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
l = json.loads(open("gpurun_out/dev_bench.json").read().strip().splitlines()[-1])
print("value", l["value"], "ms", l["ms_per_step"], "e2e", l["e2e"]["value"])
print(l["stages_ms"])
print({k: round(v["frac"], 3) for k, v in l["stage_roofline"].items() if isinstance(v, dict)})
PY
if [ -n "$NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/dev_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu list rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${NCU_KERNEL:-gate_kernel}" -c 2 -o gpurun_out/dev_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu full rc=$?"
  ncu -i gpurun_out/dev_full.ncu-rep --page raw --csv > gpurun_out/dev_full_raw.csv 2>/dev/null
  ncu -i gpurun_out/dev_full.ncu-rep --page details --csv > gpurun_out/dev_full_details.csv 2>/dev/null
fi
