# Multi-GPU config-3 bench (driver-style launch) with and without the jitter prefetch.
cd $GRAFT_REPO_ROOT
N=$(nvidia-smi -L | wc -l)
for pf in "" "--no-prefetch"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29800 bench.py --gpus $N --steps 20 --warmup 5 $pf > gpurun_out/mb_n$N$pf.json 2> gpurun_out/mb_n$N$pf.err; echo "n$N $pf rc=$?"
  python -c "import json,sys; l=json.loads(open('gpurun_out/mb_n$N$pf.json').read().strip().splitlines()[-1]); print(round(l['value']/1e6,3), round(l['ms_per_step'],4), round(l['e2e']['value']/1e6,3), l['roofline']['frac'], l['stages_ms'])"
done
