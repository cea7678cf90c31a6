timeout -s KILL 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -q --maxfail=5 2>&1 | tail -3
for f in "" "--no-pdl"; do
timeout -s KILL 200 python bench.py --no-cpu-baseline --no-composable --no-e2e --no-long --no-prefill --steps 30 $f > gpurun_out/bp.json 2> gpurun_out/bp.err; python -c "import json;d=json.load(open('gpurun_out/bp.json'));print('$f', d['value'], d['roofline']['launch_ms'])"
done
