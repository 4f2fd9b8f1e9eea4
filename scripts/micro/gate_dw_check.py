"""Compare dWg of the TMA gate-dw kernel with the cp.async one (env toggle in
separate processes) on one bf16 layer; prints summary statistics."""
import os, subprocess, sys
import numpy as np

if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    sys.path.insert(0, os.getcwd())
    from tests.test_gpu_bf16 import make_inputs, run
    T, d, f, E = int(sys.argv[2]), int(sys.argv[3]), 512, 64
    ocfg, arrs = make_inputs(T, d, f, E, 7, {})
    out = run({}, T, d, f, E, 7, arrs)
    np.save(sys.argv[4], out["dgate_w"])
    sys.exit(0)

for T, d in [(4096, 256), (8192, 2048)]:
    res = {}
    for v in ("0", "1"):
        fn = f"gpurun_out/dwg_{v}.npy"
        env = dict(os.environ, MOE_B200_GATE_DW_TMA=v)
        subprocess.run([sys.executable, __file__, "child", str(T), str(d), fn], env=env, check=True)
        res[v] = np.load(fn)
    a, b = res["0"].astype(np.float64), res["1"].astype(np.float64)
    print(T, d, "old |.|max", np.abs(a).max(), "new |.|max", np.abs(b).max(), "maxdiff", np.abs(a - b).max(),
          "zeros new", int((b == 0).sum()), "of", b.size)
    bad = np.argwhere(np.abs(a - b) > 1e-3 * np.abs(a).max())
    print(" bad count", len(bad), "first", bad[:8].tolist())
