V=$1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_synth.py tests/test_gpu_hot_window.py tests/test_gpu_regions.py tests/test_gpu_stress.py -x -q > gpurun_out/${V}_pytest_quick.log 2>&1; echo pytest_exit=$? >> gpurun_out/${V}_pytest_quick.log
for c in 2 5; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --streams 1 > gpurun_out/${V}_bench_C$c.jsonl 2> gpurun_out/${V}_bench_C$c.err; done
