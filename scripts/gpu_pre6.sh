timeout -s KILL 400 python -m pytest tests/test_gpu_tc.py tests/test_composable.py -q --maxfail=5 -k "prefill or composable" 2>&1 | tail -3
timeout -s KILL 300 python bench.py --no-cpu-baseline --no-e2e --no-composable --no-long --steps 5 --layers 4 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('v2',d['prefill']['value'],d['prefill']['ms_per_layer'])"
