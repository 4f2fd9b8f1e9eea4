# EP A/B (gpurun --gpus N): tests with the candidate switches on, then the
# config-3 bench with each combination.  AB_ENV0..3 = env assignments.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
env $AB_TEST_ENV timeout 1800 python -m pytest tests/test_gpu_ep.py -q -x 2>&1 | tail -2
for r in 1 2 3; do for e in "$AB_ENV0" "$AB_ENV1" "$AB_ENV2" "$AB_ENV3"; do
  [ -z "$e" ] && continue
  env $e timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29700 bench.py --gpus $N --steps 20 --warmup 5 2>/dev/null > gpurun_out/mab.json
  python -c "import json; l=json.loads(open('gpurun_out/mab.json').read().strip().splitlines()[-1]); print('$e', round(l['value']/1e6,3), round(l['ms_per_step'],4), {k[:12]:round(v,4) for k,v in l['stages_ms'].items() if not k.startswith('ffn')})"
done; done
