#!/bin/bash
# A/B of memory-path knobs on the synthetic configs (device-resident steps only)
# usage: entry_ab.sh "cfgs" "VAR=val;VAR=val ..." (variants separated by spaces)
cfgs=${1:-"3 5 2"}
variants=${2:-"AIWC_HOT_WINDOW=0 AIWC_HOT_WINDOW=1"}
for cfg in $cfgs; do
  for v in $variants; do
    env ${v//;/ } timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('cfg $cfg $v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phases_ms'].items()}, d.get('report_check'))"
  done
done
