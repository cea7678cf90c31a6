timeout -s KILL 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout -s KILL 600 python bench.py --no-cpu-baseline --no-e2e --no-prefill --no-long --steps 10 --layers 4 > gpurun_out/bc4.json 2> gpurun_out/bc4.err; python -c "import json;d=json.load(open('gpurun_out/bc4.json'));print(d['value'], d['composable'])"
