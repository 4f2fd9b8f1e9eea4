# Config-4 stack under EP (gpurun --gpus N): A/B of env switches, AB_ENV0..2
cd $GRAFT_REPO_ROOT
N=$(nvidia-smi -L | wc -l)
for r in 1 2; do for e in "$AB_ENV0" "$AB_ENV1" "$AB_ENV2"; do
  [ -z "$e" ] && continue
  env $e timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29750 bench.py --workload c4 --gpus $N --steps 5 --warmup 3 2>/dev/null > gpurun_out/c4ab.json
  python -c "import json; l=json.loads(open('gpurun_out/c4ab.json').read().strip().splitlines()[-1]); print('$e', round(l['value']/1e6,3), round(l['ms_per_step'],3))"
done; done
