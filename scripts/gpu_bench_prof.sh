# bench + ncu evidence for the decode kernel (round 1)
set -x
timeout 900 python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; tail -5 gpurun_out/bench_r01.err; cat gpurun_out/bench_r01.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 3 --layers 8 --no-cpu-baseline --no-e2e --no-prefill --no-graph > /dev/null 2>&1; tail -3 gpurun_out/launches_r01.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_decode -s 4 -c 1 -o gpurun_out/prof_decode_r01 python bench.py --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --no-e2e --no-prefill --no-graph > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
