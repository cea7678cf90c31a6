timeout -s KILL 1200 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_fp8_kv.py -m gpu -q -x 2>&1 | tail -2
B="--no-prefill --no-composable --no-long --no-contiguous --no-fp8 --no-cpu-baseline --no-e2e"
for i in 1 2; do
timeout -s KILL 600 python bench.py $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NEW value', round(d['value'],4), 'frac', round(d['frac_of_hbm_peak'],4), 'launch_ms', round(d['roofline']['launch_ms'],5))"
BSRA_LIB=abtmp/libbsra_old.so timeout -s KILL 600 python bench.py $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('OLD value', round(d['value'],4), 'frac', round(d['frac_of_hbm_peak'],4), 'launch_ms', round(d['roofline']['launch_ms'],5))"
done
mkdir -p /tmp/reps
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tc_decode_f8 -s 4 -c 1 -o /tmp/reps/f8 python bench.py --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --no-e2e --no-graph --no-prefill --no-composable --no-long --no-contiguous > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/reps/f8.ncu-rep 312877828 > gpurun_out/ncu_tc_decode_f8_r01s3.txt 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tc_decode_kernel -s 4 -c 1 -o /tmp/reps/dec python bench.py --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --no-e2e --no-graph --no-prefill --no-composable --no-long --no-contiguous --no-fp8 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/reps/dec.ncu-rep 623602436 > gpurun_out/ncu_tc_decode_r01s3.txt 2>&1
cat gpurun_out/ncu_tc_decode_f8_r01s3.txt gpurun_out/ncu_tc_decode_r01s3.txt | grep -E "kernel|duration|achieved|no_instr|long_score|wait "
