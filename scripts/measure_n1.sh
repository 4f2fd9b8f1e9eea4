#!/bin/bash
# One-GPU measurement set for profiles/: bench (ours + reference arm), the ncu
# launch list and one full-set capture of the dominant kernels.  Run via gpurun.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"grouped_gemm|chunk_kernel|logits_kernel|dw_kernel|dx_kernel|softmax|assign|dispatch|combine" -c 24 \
    -o gpurun_out/full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
