#!/bin/bash
# per-rank cost of the multi-GPU path at world size 1 (NCCL, AIWC_BENCH_SHARDED=1) next to the single-GPU step
V=$1; shift
for c in "$@"; do
  AIWC_SHARD_PROFILE=${PROFILE:-0} AIWC_BENCH_SHARDED=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29571 bench.py --gpus 1 --config $c --no-e2e --steps 5 > gpurun_out/${V}_sharded_C$c.jsonl 2> gpurun_out/${V}_sharded_C$c.err
done
