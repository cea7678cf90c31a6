timeout -s KILL 400 python scripts/composable_perf.py 2>&1 | tail -9
timeout -s KILL 900 python -m pytest tests/test_full_size.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_r2d.json 2> gpurun_out/bench_r2d.err; tail -2 gpurun_out/bench_r2d.err; python -c "import json;d=json.load(open('gpurun_out/bench_r2d.json'));print(d['value'], d['e2e']['value'], d['prefill']['value'], d['composable']['us_per_layer']); print(json.dumps(d['quest']))"
