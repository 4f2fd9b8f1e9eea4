# Multi-GPU session (gpurun --gpus N): EP tests + bench at N GPUs + 1 GPU with E/N experts.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_ep.py -q -rA -s > gpurun_out/pytest_ep_n$N.log 2>&1; echo "pytest ep rc=$?"
tail -5 gpurun_out/pytest_ep_n$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29600 bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "bench n$N rc=$?"
tail -c 600 gpurun_out/bench_n$N.json
