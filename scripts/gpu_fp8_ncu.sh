timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tc_decode -s 10 -c 1 -o gpurun_out/prof_fp8_decode python scripts/fp8_perf.py > gpurun_out/ncu_fp8.log 2>&1
tail -3 gpurun_out/ncu_fp8.log
