timeout -s KILL 900 python -m pytest tests/test_plan_device.py -m gpu -q -x > gpurun_out/pytest_r2p.txt 2>&1; tail -3 gpurun_out/pytest_r2p.txt; grep -E "Error|assert" gpurun_out/pytest_r2p.txt | head -5
timeout -s KILL 300 python scripts/prefill_overhead.py 2>&1 | tail -12
