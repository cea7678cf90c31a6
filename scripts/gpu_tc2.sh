timeout 600 python -m pytest tests/test_gpu_tc.py -q --maxfail=10 2>&1 | tail -30
timeout 600 python bench.py --no-cpu-baseline --no-prefill > gpurun_out/bench_tc2.json 2> gpurun_out/bench_tc2.err; tail -3 gpurun_out/bench_tc2.err; cat gpurun_out/bench_tc2.json
