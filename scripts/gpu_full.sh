timeout -s KILL 900 python -m pytest tests -m gpu -q --maxfail=10 2>&1 | tail -15
timeout -s KILL 600 python bench.py > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err; tail -3 gpurun_out/bench_r01b.err; cat gpurun_out/bench_r01b.json
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tc_prefill -s 1 -c 1 -o gpurun_out/prof_prefill_r01 python bench.py --steps 1 --warmup 3 --layers 1 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/ncu_pre.log 2>&1; tail -2 gpurun_out/ncu_pre.log
