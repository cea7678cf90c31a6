set -x
timeout 300 python -m pytest tests/test_gpu_tc.py -q -x -k basic 2>&1 | tail -30
timeout 600 python -m pytest tests/test_gpu_tc.py -q --maxfail=10 2>&1 | tail -40
