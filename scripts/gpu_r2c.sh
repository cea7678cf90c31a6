timeout -s KILL 600 compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/sanitize.py > gpurun_out/sanitize_racecheck.txt 2>&1; echo racecheck rc=$?; grep -c "Race reported" gpurun_out/sanitize_racecheck.txt
timeout -s KILL 300 python scripts/composable_perf.py 2>&1 | tail -9
timeout -s KILL 300 python -m pytest tests -m gpu -q -x -k "prefill or c3 or composable" 2>&1 | tail -2
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-long --no-contiguous --no-fp8 --no-sched --no-composable > gpurun_out/bench_r2c.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/bench_r2c.json'));print(d['value'], d['prefill']['value'], d['prefill']['ms_per_layer'])"
