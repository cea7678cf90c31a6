set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.max.mem --format=csv
timeout -s KILL 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -4
timeout -s KILL 900 python bench.py > gpurun_out/bench_r01s5.json 2> gpurun_out/bench_r01s5.err; head -c 300 gpurun_out/bench_r01s5.json
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r01s5.json 2>/dev/null; head -c 200 gpurun_out/bench_ref_r01s5.json
mkdir -p /tmp/reps
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tc_decode_f8 -s 4 -c 1 -o /tmp/reps/f8 python bench.py --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --no-e2e --no-graph --no-prefill --no-composable --no-long --no-contiguous > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/reps/f8.ncu-rep 312877828 > gpurun_out/ncu_tc_decode_f8_r01s5.txt 2>&1
head -5 gpurun_out/ncu_tc_decode_f8_r01s5.txt
