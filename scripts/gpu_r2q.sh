timeout -s KILL 900 python -m pytest tests/test_plan_device.py -m gpu -q -x > gpurun_out/pytest_r2q.txt 2>&1; tail -3 gpurun_out/pytest_r2q.txt; grep -E "Error|assert" gpurun_out/pytest_r2q.txt | head -5
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg --clock-control none -k regex:"tc_prefill|contraction" --csv --log-file gpurun_out/ncu_pre_oh.csv python scripts/prefill_overhead.py > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/ncu_pre_oh.csv')) if r and not r[0].startswith('==')]
hdr=rows[0]
for r in rows[1:]:
    d=dict(zip(hdr,r))
    if d['Metric Name']=='gpu__time_duration.sum': print(d['ID'], d['Kernel Name'][:40], d['Metric Value'])
PY
