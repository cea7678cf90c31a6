timeout -s KILL 600 python -m pytest tests/test_composable.py tests/test_sequence_split.py -q -m gpu --maxfail=5 2>&1 | tail -15
timeout -s KILL 900 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_c45.json 2> gpurun_out/bench_c45.err; tail -5 gpurun_out/bench_c45.err; cat gpurun_out/bench_c45.json
