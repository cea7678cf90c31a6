timeout -s KILL 900 python -m pytest tests/test_fp8_kv.py tests/test_gpu_tc.py -m gpu -q -x > gpurun_out/pytest_r2l.txt 2>&1; tail -2 gpurun_out/pytest_r2l.txt
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-prefill --no-sched --no-long --no-quest --no-composable --no-e2e --no-contiguous --no-rope > gpurun_out/bench_r2l.json 2> gpurun_out/bench_r2l.err; tail -2 gpurun_out/bench_r2l.err; python -c "import json;d=json.load(open('gpurun_out/bench_r2l.json'));print('decode', d['value'], d['roofline']['launch_ms'], 'fp8', d['decode_fp8']['value'], d['decode_fp8']['launch_ms'], d['decode_fp8']['speedup_vs_bf16_kv'])"
for v in base rl80 rl88 emu1 emu2; do
  if [ $v = base ]; then L=paper_2501_01005_b200/libbsra.so; else L=abtmp/libbsra_$v.so; fi
  echo "$v: $(BSRA_LIB=$L timeout -s KILL 200 python scripts/ab_prefill.py 256 2>&1 | tail -1)"
done
timeout -s KILL 600 python scripts/composable_perf.py 2>&1 | grep -v "^{" | cut -c1-150
