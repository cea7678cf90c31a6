timeout -s KILL 1200 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_variants.py tests/test_composable.py tests/test_sequence_split.py tests/test_ragged_kv.py -m gpu -q -x 2>&1 | tail -2
B="--no-prefill --no-composable --no-long --no-contiguous --no-fp8 --no-cpu-baseline --no-e2e"
for i in 1 2; do
timeout -s KILL 600 python bench.py $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NEW value', round(d['value'],4), 'frac', round(d['frac_of_hbm_peak'],4), 'launch_ms', round(d['roofline']['launch_ms'],5))"
BSRA_LIB=abtmp/libbsra_old.so timeout -s KILL 600 python bench.py $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('OLD value', round(d['value'],4), 'frac', round(d['frac_of_hbm_peak'],4), 'launch_ms', round(d['roofline']['launch_ms'],5))"
done
