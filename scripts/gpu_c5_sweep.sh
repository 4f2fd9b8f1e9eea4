#!/bin/bash
# C5 inference sweep (eval, C=2.0, d=1024, f=4096), E_k in {8, 16}, T in {4k .. 256k}.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/${TAG:-c5}_sweep.jsonl
: > $out
for E in 8 16; do for T in 4096 16384 65536 262144; do
  timeout 300 python bench.py --workload c5 --experts $E --tokens $T --steps 20 --warmup 5 --no-cpu-baseline >> $out 2>> gpurun_out/c5.err
done; done
python - $out <<'PY'
import json, sys
for l in open(sys.argv[1]):
    d = json.loads(l)
    c = d["config"]; s = d.get("stages_ms", {})
    print(c.get("experts", c.get("num_experts")), c.get("tokens", c.get("global_batch")), round(d["value"] / 1e6, 2), "M tok/s", round(d["ms_per_step"], 4), {k: round(v * 1e3, 1) for k, v in s.items() if v > 0.002})
PY
