for d in 0 16 32 48 1 2 3; do
echo "dbg=$d"; BSRA_DEBUG_PREFILL=$d timeout -s KILL 120 python scripts/ab_prefill.py 256 128
done
