for d in 8 11; do
BSRA_DEBUG_PREFILL=$d timeout -s KILL 120 python scripts/trace_prefill.py > gpurun_out/trace_pair_$d.json 2>/dev/null
echo "== dbg $d"; python scripts/trace_summary.py gpurun_out/trace_pair_$d.json
done
