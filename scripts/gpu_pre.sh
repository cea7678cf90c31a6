timeout -s KILL 120 python -m pytest tests/test_gpu_tc.py -q -x -k "prefill_masks_tiles and causal and 128" 2>&1 | tail -30
timeout -s KILL 400 python -m pytest tests/test_gpu_tc.py -q --maxfail=10 -k prefill 2>&1 | tail -30
