# End-of-round evidence on one GPU: smoke, full GPU suite, default bench, the
# reference arm, and the ncu launch list of the bench (after a clean run).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r02l}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -rA > gpurun_out/${T}_pytest_gpu_1gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${T}_pytest_gpu_1gpu.log
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu list rc=$?"
