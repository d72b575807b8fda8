set -x
python scripts/one_exact.py > gpurun_out/k4_one.txt 2>&1
ncu --set full --import-source on --clock-control none --kernel-name regex:k_exact_task_thr -c 14 -o gpurun_out/k4_full -f python scripts/one_exact.py > gpurun_out/k4_ncu.log 2>&1
