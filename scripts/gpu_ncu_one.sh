# ncu --set full of the kernels matching KREGEX in one bench step (after a clean
# bench run); writes gpurun_out/$TAG.ncu-rep and its raw / details exports.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "bench rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$KREGEX" -c ${COUNT:-4} -o gpurun_out/$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null; echo "export rc=$?"
