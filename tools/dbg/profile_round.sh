#!/bin/bash
# one GPU session: bench lines for every config, the reference arm, the C2 launch list,
# ncu --set full captures of the ingest kernel on C2 and C3 (after the runs without ncu)
cd "$(dirname "$0")/../.."
O=gpurun_out/prof
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 600 python bench.py > $O/bench_C2.jsonl 2> $O/bench_C2.err
for c in 1 3 4 5; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_C$c.jsonl 2> $O/bench_C$c.err; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_C2.jsonl 2> $O/bench_ref_C2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C2.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --streams 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ingest_kernel --launch-skip 3 --launch-count 1 \
  -o $O/ingest_C2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --streams 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ingest_kernel --launch-skip 3 --launch-count 1 \
  -o $O/ingest_C3 python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --streams 1 > /dev/null 2>&1
ls -la $O
