BSRA_LIB=$PWD/paper_2501_01005_b200/libbsra_head.so timeout -s KILL 120 python scripts/ab_prefill.py 128
timeout -s KILL 120 python scripts/ab_prefill.py 128 256
BSRA_DEBUG_PREFILL=32 timeout -s KILL 120 python scripts/ab_prefill.py 256
timeout -s KILL 120 python scripts/trace_prefill.py > gpurun_out/trace_pair_0.json 2>/dev/null
timeout -s KILL 300 python -m pytest tests/test_gpu_tc.py -q -x -k "prefill" 2>&1 | tail -2
