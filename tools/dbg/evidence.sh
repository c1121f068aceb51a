#!/bin/bash
# ncu --set full of EVERY kernel of one step per workload (after the programs ran
# without ncu), summarised ON THE BOX (reports are deleted: gpurun brings back <= 64 MiB),
# plus compute-sanitizer memcheck / racecheck on small traces.
# usage: tools/dbg/evidence.sh OUTDIR [workload ...]
cd "$(dirname "$0")/../.."
O=$1; shift
mkdir -p $O
W=${@:-C2 C3 C4 C5 validate2 sparse2 regions2 job2 sim C1}
for w in $W; do
  timeout 300 python tools/prof_step.py $w > $O/plain_$w.log 2>&1 || echo "plain $w failed" >> $O/fail.txt
  timeout 1500 ncu --set full --import-source on --clock-control none --profile-from-start off \
    -o /tmp/step_$w python tools/prof_step.py $w > $O/ncu_$w.log 2>&1 || echo "ncu $w failed" >> $O/fail.txt
  python tools/ncu_summary.py /tmp/step_$w.ncu-rep > $O/summary_$w.txt 2>&1
  ncu -i /tmp/step_$w.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread > $O/raw_$w.csv 2>&1
  rm -f /tmp/step_$w.ncu-rep
done
ls -la $O
