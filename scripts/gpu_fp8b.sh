timeout -s KILL 600 python -m pytest tests/test_fp8_kv.py -m gpu -x -q 2>&1 | tail -4
timeout -s KILL 300 python scripts/fp8_perf.py 2>&1 | tail -2
