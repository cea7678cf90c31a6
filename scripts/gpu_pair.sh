# paired 256-row prefill tile: quick parity, full prefill parity, prefill bench A/B (T_q 128 vs 256)
set -x
make -s 2>&1 | grep -i error
timeout -s KILL 120 python -m pytest tests/test_gpu_tc.py -q -x -k "prefill_masks_tiles and causal and 256" 2>&1 | tail -15
timeout -s KILL 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -q --maxfail=10 -k "prefill or tiles_masks" 2>&1 | tail -25
for t in 128 256; do
timeout -s KILL 300 python bench.py --no-cpu-baseline --no-composable --no-e2e --no-long --steps 3 --layers 2 --prefill-tile $t > gpurun_out/bp$t.json 2> gpurun_out/bp$t.err; tail -2 gpurun_out/bp$t.err; python -c "import json;d=json.load(open('gpurun_out/bp$t.json'));print($t, d['prefill'])"
done
