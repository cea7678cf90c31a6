timeout -s KILL 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
s=$(date +%s); timeout -s KILL 900 python bench.py > gpurun_out/bench_r01_final.json 2> gpurun_out/bench_r01_final.err; e=$(date +%s); echo "bench seconds: $((e-s))"; tail -3 gpurun_out/bench_r01_final.err; cat gpurun_out/bench_r01_final.json
s=$(date +%s); timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; e=$(date +%s); echo "ref seconds: $((e-s))"; tail -3 gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
