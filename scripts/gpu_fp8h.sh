timeout -s KILL 600 python -m pytest tests/test_fp8_kv.py -m gpu -q -x 2>&1 | tail -1
B="--no-prefill --no-composable --no-long --no-contiguous --no-cpu-baseline --no-e2e"
for i in 1 2; do
timeout -s KILL 600 python bench.py $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); f=d['decode_fp8']; print('NEW bf16', round(d['ms_per_step'],4), 'fp8', round(f['ms_per_step'],4), 'fp8 launch', round(f['launch_ms'],5))"
BSRA_LIB=abtmp/libbsra_old.so timeout -s KILL 600 python bench.py $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); f=d['decode_fp8']; print('OLD bf16', round(d['ms_per_step'],4), 'fp8', round(f['ms_per_step'],4), 'fp8 launch', round(f['launch_ms'],5))"
done
