timeout -s KILL 600 python scripts/composable_perf.py 2>&1 | grep -v "^{" | cut -c1-150 | tail -5
