#!/bin/bash
# Same-box interleaved A/B of the current engine against several builds:
# usage: tools/dbg/ab_multi.sh OUT "cfgs" name1 name2 ... (abl/libaiwc_NAME.so), 3 rounds
OUT=$1; CFGS=$2; shift 2
for c in $CFGS; do
  for i in 1 2 3; do
    for v in cur "$@"; do
      if [ $v = cur ]; then envs=""; else envs="AIWC_LIB=$PWD/abl/libaiwc_$v.so"; fi
      echo -n "C$c $v " >> $OUT
      env $envs timeout 300 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline --streams 1 2>&1 | \
        python -c "import json,sys
try:
  d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],4), round(d['phases_ms']['ingest'],4), round(d['phases_ms']['pass1'],4))
except Exception as e: print('ERR', e)" >> $OUT
    done
  done
done
