#!/bin/bash
# bench.py's N>1 path (config 3, SPMD) with two ranks on the one GPU; $1 = transport (host | nccl)
mkdir -p gpurun_out
T=${1:-host}
BENCH_SAME_GPU=1 BENCH_TRANSPORT=$T timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 --batch 64 \
  > gpurun_out/spmd_bench_$T.json 2> gpurun_out/spmd_bench_$T.err
