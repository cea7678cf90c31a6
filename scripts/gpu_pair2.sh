# prefill A/B: T_q 128 (streamed) vs 256 (paired), quick parity first
make -s 2>&1 | grep -i error
timeout -s KILL 300 python -m pytest tests/test_gpu_tc.py -q -x -k "prefill_masks_tiles or prefill_num_ctas" 2>&1 | tail -3
for t in 128 256; do
timeout -s KILL 300 python bench.py --no-cpu-baseline --no-composable --no-e2e --no-long --steps 3 --layers 2 --prefill-tile $t > gpurun_out/bp$t.json 2> gpurun_out/bp$t.err; tail -2 gpurun_out/bp$t.err; python -c "import json;d=json.load(open('gpurun_out/bp$t.json'));p=d['prefill'];print($t, p['value'], p['ms_per_layer'])"
done
