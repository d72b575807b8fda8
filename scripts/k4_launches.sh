# K4 launch list (config 1-B&B, third exhaustive call of time_exact.py) -> gpurun_out/k4_launches.csv
timeout 200 python scripts/time_exact.py > gpurun_out/k4_time.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k4_launches.csv \
  python scripts/one_exact.py > gpurun_out/k4_ncu.log 2>&1; echo ncu rc=$?
