#!/bin/bash
# One gpurun call: GPU tests (optionally a -k filter), smoke, and a short bench.
#   scripts/gpu_suite.sh [tag] [pytest -k expression]
tag=${1:-run}; kexpr=${2:-}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
if [ -n "$kexpr" ]; then
  timeout -s KILL 1800 python -m pytest tests -m gpu -q -x -k "$kexpr" > gpurun_out/pytest_$tag.txt 2>&1
else
  timeout -s KILL 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_$tag.txt 2>&1
fi
tail -25 gpurun_out/pytest_$tag.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -4
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
tail -3 gpurun_out/bench_$tag.err; head -c 600 gpurun_out/bench_$tag.json
