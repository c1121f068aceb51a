#!/bin/bash
# build the engine from a copy of the tree with a python patch applied: build_variant.sh NAME PATCH.py
# (measurement only; output abl/libaiwc_NAME.so)
set -e
cd "$(dirname "$0")/../.."
N=$1; P=$(realpath "$2")
D=/tmp/variant_$N
rm -rf $D && mkdir -p $D
cp -r include paper_1805_04207_b200 $D/
(cd $D && python "$P")
S=$D/paper_1805_04207_b200/csrc
mkdir -p abl
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -o abl/libaiwc_$N.so \
  $S/{aiwc_ingest,aiwc_util,aiwc_memory,aiwc_dense,aiwc_branch,aiwc_capi,aiwc_synth,aiwc_validate,aiwc_sim,aiwc_exchange,aiwc_bins}.cu -lnccl
