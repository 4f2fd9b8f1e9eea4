#!/bin/bash
# Run the N=1 bench for the in-tree library and each build/variants/<name>; print key stage times.
for v in cur "$@"; do
  if [ $v = cur ]; then unset MOE_B200_LIB; else export MOE_B200_LIB=$PWD/build/variants/$v/libmoe_b200.so; fi
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bv_$v.json 2>gpurun_out/bv_$v.err
  python - "$v" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/bv_{sys.argv[1]}.json"))
s = d["stages_ms"]
print(sys.argv[1], round(d["value"]), round(d["ms_per_step"], 4), {k: s[k] for k in s if "ffn" in k or "gate" in k or "jitter" in k})
PY
done
