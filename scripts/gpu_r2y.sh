for d in 0 64 192 1; do
  echo "dbg=$d: $(BSRA_DEBUG_PREFILL=$d BSRA_LIB=abtmp/libbsra_exp.so timeout -s KILL 200 python scripts/ab_prefill.py 256 2>&1 | tail -1)"
done
