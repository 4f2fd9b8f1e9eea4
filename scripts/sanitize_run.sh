set -x
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_layer.py (run via gpurun)
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm --format=csv
python scripts/sanitize_layer.py all > gpurun_out/san_plain.log 2>&1; echo rc=$?
for tool in memcheck racecheck synccheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_layer.py all > gpurun_out/san_$tool.log 2>&1; echo $tool rc=$?
done
tail -5 gpurun_out/san_*.log
