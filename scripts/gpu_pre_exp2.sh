for d in 0 3; do
BSRA_DEBUG_PREFILL=$d timeout -s KILL 300 python bench.py --no-cpu-baseline --no-e2e --no-composable --no-long --steps 2 --layers 2 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('dbg=$d', round(d['prefill']['ms_per_layer']*1000,1), 'us', round(d['prefill']['value'],1))"
done
BSRA_DEBUG_PREFILL=11 timeout -s KILL 200 python scripts/trace_prefill.py > gpurun_out/trace_d11.json 2> gpurun_out/trace.err
