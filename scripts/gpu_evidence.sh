#!/bin/bash
# Round evidence in one gpurun call: GPU tests, smoke, bench (both arms), the ncu launch list of
# the bench and ncu --set full summaries of the top kernels (decode, prefill, fp8 decode, the
# page-size-1 gather4 decode). Output under gpurun_out/ (tag = $1). compute-sanitizer is closed on
# this pool (the sanitizer logs under profiles/ are from earlier in the round, scripts/sanitize.py).
tag=${1:-ev}
mkdir -p gpurun_out /tmp/reps
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.max.mem --format=csv,noheader
timeout -s KILL 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_$tag.txt 2>&1; tail -2 gpurun_out/pytest_$tag.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.txt 2>&1; tail -3 gpurun_out/smoke_$tag.txt
timeout -s KILL 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -2 gpurun_out/bench_$tag.err
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$tag.json 2>/dev/null; head -c 300 gpurun_out/bench_ref_$tag.json; echo
Q="--no-cpu-baseline --no-e2e --no-long --no-contiguous --no-sched --no-quest --no-rope --no-composable"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_|contraction|merge|plan_device|f8_gather|attn_simt" -c 80 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --layers 4 $Q > /dev/null 2>&1; echo "launch list rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tc_decode_kernel -s 8 -c 1 -o /tmp/reps/dec python bench.py --steps 1 --warmup 3 --layers 2 --no-graph --no-prefill --no-fp8 $Q > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/reps/dec.ncu-rep 623602436 > gpurun_out/ncu_tc_decode_$tag.txt 2>&1; head -16 gpurun_out/ncu_tc_decode_$tag.txt
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tc_prefill2 -s 2 -c 1 -o /tmp/reps/pre python bench.py --steps 1 --warmup 3 --layers 2 --no-graph --no-fp8 $Q > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/reps/pre.ncu-rep 0 396773294080 > gpurun_out/ncu_tc_prefill_$tag.txt 2>&1; head -16 gpurun_out/ncu_tc_prefill_$tag.txt
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tc_decode_f8 -s 8 -c 1 -o /tmp/reps/f8 python bench.py --steps 1 --warmup 3 --layers 2 --no-graph --no-prefill $Q > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/reps/f8.ncu-rep 312877828 > gpurun_out/ncu_tc_decode_f8_$tag.txt 2>&1; head -12 gpurun_out/ncu_tc_decode_f8_$tag.txt
