for d in 0 1 2 3 4 5; do
BSRA_DEBUG_PREFILL=$d timeout -s KILL 300 python bench.py --no-cpu-baseline --no-e2e --no-composable --no-long --steps 2 --layers 2 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('dbg=$d', round(d['prefill']['ms_per_layer']*1000,1), 'us', round(d['prefill']['value'],1))"
done
