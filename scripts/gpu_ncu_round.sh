# Round-2 ncu evidence: launch list of the bench (2 steps) and full captures of the
# dominant kernels (row GEMM, weight-gradient GEMM, fused gate, gate backward).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG:-r02j}_bench.json 2> gpurun_out/${TAG:-r02j}_bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG:-r02j}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:grouped_gemm_kernel|gate_kernel|dx_kernel|dw_kernel|chunk_kernel|dispatch_gather|combine_kernel|combine_bwd|router_combine_bwd|round_wg" -c 18 -o gpurun_out/${TAG:-r02j}_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/${TAG:-r02j}_full.ncu-rep --page raw --csv > gpurun_out/${TAG:-r02j}_full_raw.csv 2>/dev/null; echo "export rc=$?"
