for i in 1 2; do
timeout -s KILL 300 python bench.py --no-cpu-baseline --no-prefill --no-composable --no-long --no-e2e --steps 30 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('wd  ',d['value'],d['roofline']['launch_ms'])"
BSRA_LIB=$PWD/paper_2501_01005_b200/libbsra_nowd.so timeout -s KILL 300 python bench.py --no-cpu-baseline --no-prefill --no-composable --no-long --no-e2e --steps 30 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('nowd',d['value'],d['roofline']['launch_ms'])"
done
nvidia-smi --query-gpu=name,clocks.max.mem,memory.total --format=csv
