#!/bin/bash
# Round-end evidence in one GPU call: smoke, bench lines (default + C1..C5 + the
# reference arm), the ncu launch list of the default bench command, the ingest
# kernel's DRAM traffic for C2 / C3 (profiles/ncu_traffic_C*.json), and per-kernel
# ncu summaries of one step of the given workloads.
# usage: tools/dbg/final_evidence.sh TAG [workload ...]
cd "$(dirname "$0")/../.."
V=$1; shift
O=gpurun_out/$V
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke_exit=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.jsonl 2> $O/bench_default.err
for c in 1 3 4 5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_C$c.jsonl 2> $O/bench_C$c.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.jsonl 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_C2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/launches_C2.log 2>&1
for c in 2 3; do
  timeout 1200 ncu --set full --clock-control none -k regex:ingest_kernel -c 1 -o /tmp/ing_C$c \
    python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_ing_C$c.log 2>&1
  python tools/ncu_traffic.py /tmp/ing_C$c.ncu-rep $c >> $O/ncu_ing_C$c.log 2>&1
  python tools/ncu_summary.py /tmp/ing_C$c.ncu-rep > $O/ncu_ing_summary_C$c.txt 2>&1
  rm -f /tmp/ing_C$c.ncu-rep
done
cp profiles/ncu_traffic_C2.json profiles/ncu_traffic_C3.json $O/ 2>/dev/null
if [ $# -gt 0 ]; then bash tools/dbg/evidence.sh $O/steps "$@"; fi
ls -la $O
