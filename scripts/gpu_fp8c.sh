timeout -s KILL 300 python scripts/fp8_perf.py 2>&1 | tail -1
BSRA_DEBUG_DECODE=8 timeout -s KILL 300 python scripts/fp8_perf.py 2>&1 | tail -1
