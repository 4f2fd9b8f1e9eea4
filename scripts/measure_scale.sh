#!/bin/bash
# Multi-GPU set (run via gpurun --gpus N): GPU tests incl. EP parity, then the
# bench at 1, 2, ... N GPUs (torchrun, one process per GPU, NCCL).
NG=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for n in 1 2 4 8; do
  [ $n -gt $NG ] && break
  if [ $n -eq 1 ]; then
    python bench.py --no-cpu-baseline > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
  else
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 \
      bench.py --gpus $n > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
  fi
  python -c "import json;d=json.loads(open('gpurun_out/bench_n$n.json').read().strip().splitlines()[-1]);print($n, d['value'], d['ms_per_step'], d['e2e']['value'])"
done
