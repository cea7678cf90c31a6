timeout -s KILL 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout -s KILL 120 python scripts/ab_prefill.py 128 256
