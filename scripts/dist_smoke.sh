#!/bin/bash
# Multi-process bench paths on a one-GPU box: 2 torchrun ranks share cuda:0 with a gloo
# control plane (SC_BENCH_SINGLE_DEVICE=1; throughputs are not meaningful here, the code
# paths are: frame sharding, band sharding with CUDA-IPC gather and per-frame rebalancing).
cd "$(dirname "$0")/.."
export SC_BENCH_SINGLE_DEVICE=1
for sh in frames bands; do
  timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29511 bench.py --gpus 2 --steps 6 --warmup 3 --no-cpu-baseline --shard $sh \
      > gpurun_out/dist_$sh.json 2> gpurun_out/dist_$sh.err
  echo "$sh rc=$?"; tail -c 300 gpurun_out/dist_$sh.json
done
