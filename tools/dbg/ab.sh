#!/bin/bash
# A/B of the ingest knobs on one config: bins (AIWC_BINS) x in-pass stream checks
V=$1; C=$2
for b in 1 0; do
  for chk in "" "--no-stream-check"; do
    AIWC_BINS=$b timeout 600 python bench.py --config $C --no-e2e --streams 1 --steps 5 $chk > gpurun_out/${V}_C${C}_bins${b}${chk:+_nochk}.json 2>&1
  done
done
