bash scripts/gpu_sanitize.sh
timeout -s KILL 300 python scripts/layout_perf.py 2>&1 | tail -8
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; tail -3 gpurun_out/bench_r2b.err; head -c 300 gpurun_out/bench_r2b.json
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_composable.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-prefill --no-long --no-contiguous --no-fp8 --no-sched --layers 1 > /dev/null 2>&1; echo ncu rc=$?
