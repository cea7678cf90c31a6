for ps in 16 32 64 128; do for d in 0 3; do
echo "dbg=$d"; PAGE=$ps BSRA_DEBUG_PREFILL=$d timeout -s KILL 120 python scripts/ab_prefill.py 256
done; done
