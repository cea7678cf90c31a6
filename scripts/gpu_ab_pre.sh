for i in 1 2; do
BSRA_LIB=$PWD/paper_2501_01005_b200/libbsra_head.so timeout -s KILL 120 python scripts/ab_prefill.py 128
timeout -s KILL 120 python scripts/ab_prefill.py 128 256
done
