timeout -s KILL 300 python scripts/exp_page_size.py 2>&1 | tail -5
BSRA_DEBUG_PREFILL=3 timeout -s KILL 300 python scripts/exp_page_size.py 2>&1 | tail -5
