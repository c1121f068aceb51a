#!/bin/bash
# in-pass stream check cost by part (measurement builds in abl/): 32 mask rules, 64 payload rules, 128 begin bitmap
for v in base 32 64 128 224; do
  if [ $v = base ]; then envs=""; else envs="AIWC_LIB=$PWD/abl/libaiwc_abl$v.so"; fi
  env $envs timeout 300 python bench.py --config 2 --steps 5 --no-e2e --no-cpu-baseline --streams 1 > gpurun_out/abl_check_$v.json 2>&1
done
