set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 600 python -m pytest tests/test_fp8_kv.py -m gpu -x -q 2>&1 | tail -15
timeout -s KILL 300 python scripts/fp8_perf.py 2>&1 | tail -3
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
