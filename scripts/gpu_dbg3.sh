for d in 0 64 128 192; do
BSRA_DEBUG_PREFILL=$d timeout -s KILL 120 python scripts/trace_prefill.py > gpurun_out/trace_e_$d.json 2>/dev/null
BSRA_DEBUG_PREFILL=$d timeout -s KILL 120 python scripts/ab_prefill.py 256
done
