timeout -s KILL 600 python -m pytest tests/test_rope.py -m gpu -q -x 2>&1 | tail -2
for rep in 1 2 3; do
  echo "main: $(timeout -s KILL 200 python scripts/ab_prefill.py 128 256 2>&1 | tail -2 | tr '\n' ' ')"
  echo "emu1: $(BSRA_LIB=abtmp/libbsra_emu1.so timeout -s KILL 200 python scripts/ab_prefill.py 256 2>&1 | tail -1)"
done
