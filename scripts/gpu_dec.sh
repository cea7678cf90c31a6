timeout -s KILL 400 python -m pytest tests/test_gpu_tc.py -q --maxfail=5 -k "decode" 2>&1 | tail -3
timeout -s KILL 300 python bench.py --no-cpu-baseline --no-prefill --no-composable --no-long --steps 30 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('dec',d['value'],d['roofline']['launch_ms'], d['e2e']['value'])"
