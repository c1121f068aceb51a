#!/bin/bash
# ncu --set full of EVERY kernel of one step per workload (after the programs ran
# without ncu), plus compute-sanitizer memcheck / racecheck on small traces
cd "$(dirname "$0")/../.."
O=gpurun_out/ev; mkdir -p $O
for w in C2 C4 C5 validate2 sparse2 regions2 job2 sim C1; do
  timeout 300 python tools/prof_step.py $w > $O/plain_$w.log 2>&1 || echo "plain $w failed" >> $O/fail.txt
  timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
    -o $O/step_$w python tools/prof_step.py $w > $O/ncu_$w.log 2>&1 || echo "ncu $w failed" >> $O/fail.txt
done
timeout 1200 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -o $O/step_C3 python tools/prof_step.py C3 > $O/ncu_C3.log 2>&1 || echo "ncu C3 failed" >> $O/fail.txt
ls -la $O
