# 4-GPU session: EP tests at 4 ranks, config-3 bench at N=2/4, config 4 (18-layer stack) under EP at N=1/2/4.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests/test_gpu_ep.py -q -rA -s > gpurun_out/pytest_ep_n$N.log 2>&1; echo "pytest ep rc=$?"; tail -3 gpurun_out/pytest_ep_n$N.log
out=gpurun_out/multi_n$N.jsonl
: > $out
for n in 2 4; do
  [ $n -le $N ] || continue
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700+n)) bench.py --gpus $n --steps 20 --warmup 5 >> $out 2>> gpurun_out/multi.err; echo "c3 n$n rc=$?"
done
timeout 600 python bench.py --workload c4 --steps 5 --warmup 3 >> $out 2>> gpurun_out/multi.err; echo "c4 n1 rc=$?"
for n in 2 4; do
  [ $n -le $N ] || continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29710+n)) bench.py --workload c4 --gpus $n --steps 5 --warmup 3 >> $out 2>> gpurun_out/multi.err; echo "c4 n$n rc=$?"
done
wc -l $out
