# round-1 evidence: GPU tests, smoke, default bench, ncu launch list + full captures
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.max.mem --format=csv
timeout -s KILL 1200 python -m pytest tests -m gpu -q 2>&1 | tail -5
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
/usr/bin/time -v timeout -s KILL 900 python bench.py > gpurun_out/bench_r01_final.json 2> gpurun_out/bench_r01_final.err; grep -E "Elapsed|Maximum resident" gpurun_out/bench_r01_final.err; cat gpurun_out/bench_r01_final.json
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/ncu_launches_r01.csv python bench.py --steps 2 --warmup 3 --layers 4 --no-cpu-baseline --no-e2e --no-graph --no-composable --no-long > /dev/null 2>&1; tail -4 gpurun_out/ncu_launches_r01.csv
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tc_decode -s 4 -c 1 -o gpurun_out/prof_decode_final python bench.py --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --no-e2e --no-graph --no-prefill --no-composable --no-long > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tc_prefill2 -s 1 -c 1 -o gpurun_out/prof_prefill_final python bench.py --steps 1 --warmup 3 --layers 1 --no-cpu-baseline --no-e2e --no-graph --no-composable --no-long > /dev/null 2>&1
ls -la gpurun_out/
