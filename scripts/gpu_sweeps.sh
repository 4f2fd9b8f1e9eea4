# One-GPU sweeps (gpurun): EP-overhead baselines, the other BASELINE configs, the C5 sweep,
# and the reference arm's affine-fit cross-check (host CPU).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/sweeps.jsonl
: > $out
for E in 32 16 8; do
  timeout 300 python bench.py --experts $E --steps 20 --warmup 5 --no-cpu-baseline >> $out 2>> gpurun_out/sweeps.err
done
for W in c1 c2 c4; do timeout 600 python bench.py --workload $W --steps 10 --warmup 3 >> $out 2>> gpurun_out/sweeps.err; done
for E in 8 16; do for T in 4096 16384 65536 262144; do
  timeout 300 python bench.py --workload c5 --experts $E --tokens $T --steps 20 --warmup 5 >> $out 2>> gpurun_out/sweeps.err
done; done
wc -l $out
free -g | head -2; nproc
if [ -z "$NO_FIT" ]; then timeout 1500 python scripts/ref_affine_fit.py --out gpurun_out/r02_reference_fit.json > gpurun_out/ref_fit.log 2>&1; echo "fit rc=$?"; tail -5 gpurun_out/ref_fit.log; fi
