#!/bin/bash
cd "$(dirname "$0")/../.."
for cfg in ${1:-2 3}; do
  for v in ${ABL_VARIANTS:-base 1 2 4 8 16 e64}; do
    if [ $v = base ]; then envs=""; elif [ $v = e64 ]; then envs="AIWC_DENSE_ENTRY=64"; else envs="AIWC_LIB=$PWD/abl/libaiwc_abl$v.so"; fi
    env $envs timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); print('cfg $cfg abl $v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phases_ms'].items() if k in ('pass1','ingest','memory')})
except Exception as e: print('cfg $cfg abl $v failed', e)"
  done
done
