for rep in 1 2; do
for v in main nopf; do
  if [ $v = main ]; then L=paper_2501_01005_b200/libbsra.so; else L=abtmp/libbsra_$v.so; fi
  echo "$v: $(BSRA_LIB=$L timeout -s KILL 200 python scripts/ab_prefill.py 256 2>&1 | tail -1)"
done
done
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-long --no-contiguous --no-sched --no-rope --no-composable --no-fp8 > gpurun_out/bench_r2s.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/bench_r2s.json'));print(d['value'], d['prefill']['value'], d['prefill']['ms_per_layer']); print(json.dumps(d['quest']))"
