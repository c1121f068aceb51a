#!/bin/bash
# Same-box A/B of the current engine against another build (AIWC_LIB), interleaved:
# usage: tools/dbg/ab_lib.sh OTHER.so OUT CONFIG... (each config 3 x 2 runs)
O=$1; OUT=$2; shift 2
for c in "$@"; do
  for i in 1 2 3; do
    for v in cur other; do
      if [ $v = cur ]; then envs=""; else envs="AIWC_LIB=$O"; fi
      echo -n "C$c $v " >> $OUT
      env $envs timeout 300 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline --streams 1 2>&1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],4), round(d['phases_ms']['ingest'],4))" >> $OUT
    done
  done
done
