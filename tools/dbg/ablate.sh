#!/bin/bash
# build measurement-only ablation variants of the engine into abl/ (never the product)
set -e
cd "$(dirname "$0")/../.."
mkdir -p abl
for v in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -DAIWC_ABL=$v \
    -o abl/libaiwc_abl$v.so paper_1805_04207_b200/csrc/{aiwc_ingest,aiwc_util,aiwc_memory,aiwc_dense,aiwc_branch,aiwc_capi,aiwc_synth,aiwc_validate,aiwc_sim,aiwc_exchange,aiwc_bins}.cu -lnccl &
done
wait
